"""Per-source-line warp stall samples from an ncu report (needs -lineinfo and
--import-source on at capture time).

    python tools/ncu_lines.py report.ncu-rep [--top 30]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
per = defaultdict(lambda: [0.0, defaultdict(float), ""])
path = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iS = 4
        stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) <= iS or not r[0]:
        continue
    try:
        s = float(r[iS] or 0)
    except ValueError:
        continue
    e = per[(path, int(r[0]))]
    e[0] += s
    e[2] = r[1]
    for i in stalls:
        try:
            e[1][hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(e[0] for e in per.values()) or 1.0
for (f, ln), e in sorted(per.items(), key=lambda kv: -kv[1][0])[: a.top]:
    top = sorted(e[1].items(), key=lambda kv: -kv[1])[:2]
    why = ", ".join(f"{k} {v / max(e[0], 1) * 100:.0f}%" for k, v in top)
    print(f"{e[0] / tot * 100:5.1f}%  {f}:{ln:<5} {e[2].strip()[:70]:<70}  [{why}]")
