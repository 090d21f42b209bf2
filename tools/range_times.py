"""Per-rank work of the N-GPU partition, measured one range at a time on one
GPU: each rank of `bench.py --gpus N` computes exactly its partition_by_ops
range with no dependence on the others, so the max over ranges of the range
product time is that step's compute critical path (the gather is added
separately).  Device-resident operands, CUDA events, L2 flushed between runs,
plan (select_grid + O_k + range pair counts) done once, as in bench.py.

    python tools/range_times.py [--config fateman30] [--ns 1,2,4,8] [--reps 5]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1303_7425_b200 import benchpolys  # noqa: E402
from paper_1303_7425_b200.cluster import plan_all_ranks, rebalance  # noqa: E402
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device  # noqa: E402
from paper_1303_7425_b200.parmul import Operand, count_below  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="fateman30")
ap.add_argument("--ns", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--phases", action="store_true")
ap.add_argument("--rebalance", type=int, default=2, help="rounds of cost rebalancing after the pair split")
a = ap.parse_args()
f, g = benchpolys.CONFIGS[a.config](int)
dev = torch.device("cuda", 0)
A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
st = torch.cuda.current_stream()
flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
out = {"config": a.config, "pairs": f.n * g.n, "ranks": {}}
def measure(plan, n, label):
    times, terms = [], []
    for r, (lo, hi) in enumerate(plan.ranges):
        pairs = 0
        ts = []
        for k in range(2 + a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            res = mul_on_device(A, B, f.layout, lo=lo, hi=hi, stream=st.cuda_stream, range_pairs=pairs)
            e1.record(st)
            e1.synchronize()
            pairs = res.pairs
            if k >= 2:
                ts.append(e0.elapsed_time(e1))
            nt = res.n
            res.free()
        times.append(statistics.median(ts))
        terms.append(nt)
        if a.phases:
            flush.zero_()
            res = mul_on_device(A, B, f.layout, lo=lo, hi=hi, stream=st.cuda_stream, range_pairs=pairs,
                                timing=True)
            print(f"  N={n} r={r} terms={res.n} pairs={res.pairs} " +
                  " ".join(f"{k}={v:.3f}" for k, v in res.phases.items()), flush=True)
            res.free()
    rec = {"range_ms": [round(t, 3) for t in times], "max_ms": max(times), "mean_ms": statistics.mean(times),
           "terms": terms, "loads": list(plan.plan.loads())}
    print(f"N={n} {label}: max {max(times):.3f} ms  mean {statistics.mean(times):.3f} ms  ranges {rec['range_ms']}",
          flush=True)
    return rec, times


for n in [int(x) for x in a.ns.split(",")]:
    plan = plan_all_ranks(f, g, 64, n, lambda x, y, b: count_below(x, y, b))
    rec, times = measure(plan, n, "pairs")
    out["ranks"][n] = {"by_pairs": rec}
    if n > 1 and a.rebalance:
        for it in range(a.rebalance):
            plan = rebalance(plan, times)
            rec, times = measure(plan, n, f"rebalanced x{it + 1}")
        out["ranks"][n]["rebalanced"] = rec
print(json.dumps(out))
