"""profiles/dram_bytes.json from ncu launch lists (tools/prof_all.sh): for each
benched config, the DRAM bytes (read + write) of every kernel over one
product, as ncu measured them.  bench.py reports the dominant kernel's entry
as roofline.traffic.

    python tools/dram_bytes.py gpurun_out/prof profiles/dram_bytes.json "r02"
"""
import contextlib
import gzip
import io
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import launch_summary  # noqa: E402


def main(src, dst, tag):
    out = json.loads(Path(dst).read_text()) if Path(dst).exists() else {}
    for f in sorted(Path(src).glob("launches_*_*.csv.gz")):
        cfg, coeff = f.name[len("launches_"):-len(".csv.gz")].rsplit("_", 1)
        tmp = Path(src) / (f.name[:-3])
        tmp.write_bytes(gzip.decompress(f.read_bytes()))
        with contextlib.redirect_stdout(io.StringIO()):
            agg = launch_summary.main(str(tmp), "")
        tmp.unlink()
        out[f"{cfg}/{coeff}"] = {
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({tag}): one product, "
                      f"profiles/{tag}_launches_{cfg}_{coeff}_summary.txt",
            "kernels": {name: {"launches": n, "dram_bytes": r + w, "ms": t / 1e6}
                        for name, (n, t, r, w) in agg.items()}}
    Path(dst).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "r02")
