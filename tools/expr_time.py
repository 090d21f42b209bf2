"""Time building benchmark operands from the reference's expressions on the GPU."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1303_7425_b200.expr import bench_pair
for ex, p in [(1, 30), (2, 12), (2, 25)]:
    t0 = time.perf_counter(); f, g = bench_pair(ex, p); t1 = time.perf_counter()
    print(f"example {ex} power {p}: {f.n}+{g.n} terms in {1e3*(t1-t0):.0f} ms")
