"""The reference's benchmark entry point on the GPU: SURVEY 8(f) row 3.

Mirrors the `/bench` handler (reference service/app.py:38-45, 139-167) and
its request/response models (service/models.py:54-80) as a plain function,
without the HTTP service (out of scope): the same three examples, the same
power cap, one row per (merger, threads, repetition) with the wall time of
`mul(f, g, cfg)` in milliseconds, and `verified` = product == naive_mul(f, g)
below verify_limit pairwise products.

Differences, all result-preserving: operands are built by powering with the
GPU `mul` (order-exact for f64, so float operands match the reference's bit
for bit), `threads` and `merger` are recorded but do not change the GPU
product (every merger and worker count gives the same result), and
f64 products use the order-exact fold so the result equals the reference's.

    python -m paper_1303_7425_b200.benchharness --example 2 --scale 12
prints the same `key=value` lines as the reference's `polymul bench`
(cli.py:114-138).
"""

from __future__ import annotations

import argparse
import time

from .core import naive_mul
from .expr import BENCH_EXAMPLES, bench_pair
from .parmul import MERGERS, MulConfig, mul

BENCH_POWER_CAP = 12  # without `full`, powers stay at desk scale (app.py:44-45)


class BenchInputError(ValueError):
    """Request rejected before any work (the service's HTTP 400, kind "parse")."""


def run_bench(example: int, power: int = 8, l: int = 64, threads=(1,), mergers=("heap",),
              repetitions: int = 1, coeff: str = "int", full: bool = False,
              verify_limit: int = 10 ** 6, device: int = 0) -> dict:
    """Body of a BenchResponse (models.py:66-80) for a BenchRequest."""
    if example not in BENCH_EXAMPLES:
        raise BenchInputError(f"example must be one of {sorted(BENCH_EXAMPLES)}, got {example}")
    if power < 1 or l < 1 or repetitions < 1 or not threads or not mergers:
        raise BenchInputError("power, l, repetitions >= 1 and non-empty threads/mergers required")
    if coeff not in ("int", "f64"):
        raise BenchInputError(f"coeff must be 'int' or 'f64', got {coeff!r}")
    for m in mergers:
        if m not in MERGERS:
            raise BenchInputError(f"unknown merger {m!r}")
    if not full and power > BENCH_POWER_CAP:
        raise BenchInputError(f"power {power} needs the full flag (desk-scale cap is {BENCH_POWER_CAP})")
    ctype = float if coeff == "f64" else int
    ordered = ctype is float
    build_cfg = MulConfig(float_ordered=ordered, device=device)
    f, g = bench_pair(example, power, ctype, mul=lambda a, b: mul(a, b, build_cfg))
    rows = []
    product = None
    for merger in mergers:
        for t in threads:
            cfg = MulConfig(l=l, c=int(t), merger=merger, float_ordered=ordered, device=device)
            for rep in range(repetitions):
                t0 = time.perf_counter()
                product = mul(f, g, cfg)
                rows.append({"merger": merger, "threads": int(t), "repetition": rep,
                             "time_ms": (time.perf_counter() - t0) * 1000.0})
    verified = None
    if f.n * g.n <= verify_limit:
        verified = product == naive_mul(f, g)
    return {"example": example, "power": power, "f_terms": f.n, "g_terms": g.n,
            "result_terms": product.n, "rows": rows, "verified": verified}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--example", type=int, default=1, choices=sorted(BENCH_EXAMPLES))
    ap.add_argument("--scale", type=int, default=8)
    ap.add_argument("--l", type=int, default=64)
    ap.add_argument("--threads", default="1")
    ap.add_argument("--merger", default="heap")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--coeff", default="int", choices=("int", "f64"))
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args(argv)
    body = run_bench(args.example, args.scale, args.l, [int(t) for t in args.threads.split(",")],
                     args.merger.split(","), args.reps, args.coeff, args.full)
    for key in ("example", "power", "f_terms", "g_terms", "result_terms", "verified"):
        print(f"{key}={body[key]}")
    for row in body["rows"]:
        print(f"merger={row['merger']} threads={row['threads']} "
              f"rep={row['repetition']} time_ms={row['time_ms']:.3f}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
