"""Wall time of the public API calls (host lists in, Polynomial out) vs arrays."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1303_7425_b200 import benchpolys, mul, mul_arrays, io
for name in sys.argv[1:] or ["fateman30", "mp12"]:
    f, g = benchpolys.CONFIGS[name](int)
    for k in range(3):
        t0 = time.perf_counter(); p = mul(f, g); t1 = time.perf_counter()
        q = mul_arrays(f, g); t2 = time.perf_counter()
        d = io.text_digest(q); t3 = time.perf_counter()
    print(f"{name}: mul() {1e3*(t1-t0):.1f} ms ({p.n} terms), mul_arrays() {1e3*(t2-t1):.1f} ms, "
          f"GPU PolyFile digest {1e3*(t3-t2):.1f} ms")
