"""Products on every device path, checked against the oracle (test
infrastructure only): Fateman n=6 and Monagan-Pearce n=4, int and float, and
(with --golden) every golden case, through the dense, bucket, sort and small
paths.  Run by tests/test_gpu_checked.py on the checked library (PGPU_LIB =
lib/libpolymul_b200_checked.so: device bounds assertions) and, where the pool
allows it, under compute-sanitizer."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from oracle import oracle  # noqa: E402
from paper_1303_7425_b200 import MulConfig, benchpolys, mul  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
paths = args[0].split(",") if args else ["dense", "bucket", "sort", "small"]
n = 0
for name, (f, g) in (("F6", benchpolys.fateman(6)), ("MP4", benchpolys.monagan_pearce(4)),
                     ("F6f", benchpolys.fateman(6, float)), ("MP3f", benchpolys.monagan_pearce(3, float))):
    want = oracle.mul(f, g)
    for path in paths:
        if path == "dense" and name.startswith("MP"):
            continue  # sparse key span: the dense path refuses
        if path == "small" and f.n * g.n > 16384:
            continue
        ordered = None if path != "dense" else False
        p = mul(f, g, MulConfig(path=path, float_ordered=ordered))
        assert p.exps == want.exps, (name, path)
        if f.ctype is int or ordered is None:
            assert p.coeffs == want.coeffs, (name, path)
        n += 1
if "--golden" in sys.argv:
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from conftest import golden_cases, product_digest  # noqa: E402
    from paper_1303_7425_b200.split import SplitSet  # noqa: E402
    for name, a, b, split, want in golden_cases():
        for path in paths:
            sp = None if split is None else SplitSet(split)
            try:
                p = mul(a, b, MulConfig(path=path, float_ordered=None if path != "dense" else False), split=sp)
            except Exception as exc:
                # the dense path refuses wide key spans (and ordered floats)
                assert path == "dense" and "dense path" in str(exc), (name, path, exc)
                continue
            if a.ctype is int or path != "dense":  # (dense fast floats: within tolerance only)
                assert p.n == want["n"], (name, path)
                assert product_digest(p.exps, p.coeffs) == want["sha256"], (name, path)
            n += 1
from paper_1303_7425_b200 import _native  # noqa: E402
print(f"checked run ok: {n} products ({_native.load()._name})")
