"""Per-launch summary of an ncu launch list (gpu__time_duration + dram bytes)
for the LAST product in the capture (tools/prof_step.py runs a warm-up product
first).  usage: python tools/launch_summary.py launches.csv "title" > summary.txt"""
import csv
import sys
from collections import OrderedDict


def main(path, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ids = list(launches)
    # the last product starts at the last k_stats launch pair
    starts = [i for i in ids if launches[i]["name"].startswith("void k_stats")]
    first = starts[-2] if len(starts) >= 2 else ids[0]
    sel = [launches[i] for i in ids if i >= first]
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in sel)
    print(f"# {title}")
    print(f"# one product, ncu launch list (cold-cache, serialised: compare shares, not absolutes)")
    print(f"# step total {tot / 1e6:.3f} ms over {len(sel)} launches")
    agg = OrderedDict()
    for d in sel:
        t = d.get("gpu__time_duration.sum", 0)
        if len(sel) <= 80:
            print(f"{d['name'][:70]:70s} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  dram r "
                  f"{d.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB w {d.get('dram__bytes_write.sum', 0) / 1e6:9.1f} MB")
        name = d["name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    print("# per kernel (all launches of the product)")
    for name, (n, t, r, w) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} x{n:<4d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  dram {(r + w) / 1e6:10.1f} MB "
              f"({(r + w) / max(t, 1):8.1f} GB/s)")
    return agg


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
