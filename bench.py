#!/usr/bin/env python
"""bench.py -- term products/sec of one sparse polynomial product on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config fateman30] [--coeff int|float]

A step is one full product a*b (BASELINE.json metric: Fateman n=30 f*(f+1),
46,376 x 46,376 terms, 2,150,733,376 term products; exact integer
coefficients as in the reference's default ctype).  Synthetic operands are
built in closed form (identical to the reference's poly_from_expr output).

Our arm (`--impl ours`):
  value     term products/s with both operands resident in HBM when the timed
            region starts (pgpu_mul on device buffers, result left in HBM),
            CUDA events on the launching stream, L2 flushed between steps;
  e2e       the same metric through the C ABI with pinned host buffers: H2D of
            the operands and D2H of the result inside the timed region;
  roofline  dominant kernel (numeric pass) duration from live CUDA events;
            algorithmic bytes = 32 B per term product;
  cpu_baseline  the oracle (C port of the reference algorithm) on all host
            threads over a sampled subset of the intervals (rank 0, N=1).
For N>1 (torchrun, one rank per GPU) each rank computes its partition_by_ops
range and the disjoint slices are all-gathered over NCCL; time = max over ranks.

Reference arm (`--impl reference`): the CPU implementation of the path --
the oracle port, since the reference is pure Python and does not travel --
on all host threads, each step a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "term products/sec (Fateman n=30 f*(f+1))"
UNIT = "term_products/s"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="fateman30",
                    help="workload: fateman10 | fateman20 | fateman30 | mp12 | mp25 (BASELINE.json configs)")
    ap.add_argument("--coeff", choices=["int", "float"], default="int")
    ap.add_argument("--path", default="auto",
                    help="device algorithm: auto | dense | bucket | sort | small (pgpu_options.path)")
    ap.add_argument("--gather", default="peer", choices=("peer", "collective"),
                    help="N>1: assemble the slices by peer copies (CUDA IPC) or an all-gather")
    ap.add_argument("--flush-mib", type=int, default=512)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostic only: no L2 flush between steps")
    ap.add_argument("--emulate-ranks", action="store_true",
                    help="diagnostic: run the N>1 partition/gather path with gloo, every rank on "
                         "cuda:0 (correctness only; timings are not meaningful)")
    ap.add_argument("--clock-sampler", choices=["nvml", "nvidia-smi", "none"], default="nvml")
    ap.add_argument("--verify", action="store_true",
                    help="check the assembled product against the reference digest")
    return ap.parse_args()


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class NvmlClocks:
    """In-process NVML sampling (SM clock, max clock, throttle reasons) during
    the timed region, on a background thread; lighter than spawning nvidia-smi."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.01):
        self.index = index
        self.period = period_s
        self.samples = []
        self.stop_ev = None
        self.th = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.stop_ev = threading.Event()

        def run():
            while not self.stop_ev.is_set():
                try:
                    sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                    rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
                self.stop_ev.wait(self.period)

        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def stop(self):
        if self.nv is None or self.th is None:
            return None
        self.stop_ev.set()
        self.th.join(timeout=2)
        if not self.samples:
            return None
        reasons = sorted({k for _, rs in self.samples for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.mx,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = [ln.split(",") for ln in Path(self.f.name).read_text().splitlines() if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def operands(args):
    from paper_1303_7425_b200 import benchpolys
    ct = float if args.coeff == "float" else int
    return benchpolys.CONFIGS[args.config](ct)


def workload_name(args, f, g):
    return (f"{args.config} f*g ({f.n}x{g.n} terms), "
            f"{'exact int' if args.coeff == 'int' else 'f64'} coefficients")


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(f, g, seconds_target, threads):
    """Oracle on every stride-th interval of select_grid(l=64); returns
    (pairs/s, description, pairs, seconds)."""
    from oracle import oracle as O
    bounds = O.select_grid(f, g, 64)
    P = f.n * g.n
    per_thread_rate = 4.0e6  # products/s/thread of the C heap merge (measured here)
    stride = max(1, int(P / (threads * per_thread_rate * seconds_target)))
    pairs = O.sample_pairs(f, g, bounds, stride)
    t0 = time.perf_counter()
    O.mul_raw(f, g, threads=threads, bounds=bounds, stride=stride)
    dt = time.perf_counter() - t0
    desc = (f"every {stride}th of {len(bounds) - 1} select_grid(l=64) intervals "
            f"({pairs} of {P} term products), C heap_merge port, {threads} threads")
    return pairs / dt, desc, pairs, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    f, g = operands(args)
    threads = cpu_threads()
    vals = []
    desc = ""
    for k in range(args.warmup + args.steps):
        v, desc, pairs, dt = cpu_sample(f, g, 4.0, threads)
        if k >= args.warmup:
            vals.append((pairs, dt))
    tp = sum(p for p, _ in vals)
    tt = sum(d for _, d in vals)
    value = tp / tt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tt / max(1, len(vals)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64" if args.coeff == "int" else "f64", "data": "synthetic (closed form)",
            "impl": "reference",
            "config": {"workload": workload_name(args, f, g), "sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def verify_product(args, f, step, gathered, world, rank):
    """sha256 of the reference text format of the (assembled) product vs the
    reference's recorded digest (tests/golden/digests.json)."""
    import numpy as np
    from paper_1303_7425_b200 import io
    from paper_1303_7425_b200.core import Polynomial
    from paper_1303_7425_b200.parmul import limbs_to_ints
    want = json.loads((ROOT / "tests" / "golden" / "digests.json").read_text())["products"]
    key = f"{args.config}/{args.coeff}"
    r = step()
    if world > 1:
        e, c = gathered[0]
        exps = e.cpu().numpy().view(np.uint64)
        words = c.cpu().numpy().view(np.uint64)
    else:
        e, c = r.tensors()
        exps = e.cpu().numpy().view(np.uint64)
        words = c.cpu().numpy().view(np.uint64).reshape(exps.shape[0], -1)
    if r is not None:
        r.free()
    if args.coeff == "float":
        co = words.reshape(-1).view(np.float64).tolist()
    else:
        co = limbs_to_ints(words, words.shape[1])
    p = Polynomial._from_sorted(f.layout, exps.tolist(), co, float if args.coeff == "float" else int)
    got = io.poly_digest(p)
    ok = key in want and want[key]["sha256"] == got
    return {"digest": got, "reference_digest": want.get(key, {}).get("sha256"), "ok": ok, "terms": p.n}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1303_7425_b200 import MulConfig, _native
    from paper_1303_7425_b200.cluster import plan_for_ranks, rank_range, gather_slices
    from paper_1303_7425_b200.core import SENTINEL
    from paper_1303_7425_b200.device import DeviceOperand, mul_host_pinned, mul_on_device
    from paper_1303_7425_b200.parmul import Operand, count_below

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.emulate_ranks else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.emulate_ranks:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    _native.load()

    f, g = operands(args)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    dA, dB = DeviceOperand(A, dev), DeviceOperand(B, dev)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # partition (paper Alg. 2): planned once per operand pair, timed separately
    t0 = time.perf_counter()
    lo, hi = 0, SENTINEL
    if world > 1:
        bounds, plan = plan_for_ranks(f, g, 64, world, rank,
                                      lambda x, y, b: count_below(x, y, b, device=local), None)
        lo, hi = rank_range(bounds, plan, rank)
    plan_ms = 1e3 * (time.perf_counter() - t0)

    total_pairs = f.n * g.n

    def step(timing=False):
        if lo >= hi:
            res = None
        else:
            res = mul_on_device(dA, dB, f.layout, lo=lo, hi=hi, path=args.path, device=local,
                                stream=sptr, timing=timing)
        if world > 1:
            if res is not None:
                e, c = res.tensors()
                c = c.view(torch.int64).reshape(e.shape[0], -1)
            else:
                e = torch.zeros(0, dtype=torch.int64, device=dev)
                c = torch.zeros((0, 3), dtype=torch.int64, device=dev)
            if peer[0] is not None:
                gathered[0] = peer[0].gather(e, c, stream=sptr)
            else:
                gathered[0] = gather_slices(e, c)
        return res

    gathered = [None]
    # final gather of disjoint slices: peer copies over NVLink (CUDA IPC), or
    # NCCL / gloo all-gather with --gather collective
    peer = [None]
    gather_kind = "none"
    if world > 1:
        gather_kind = args.gather
        if args.gather == "peer":
            from paper_1303_7425_b200.cluster import PeerGather
            peer[0] = PeerGather(device=local)

    flush = torch.empty(args.flush_mib * (1 << 20) // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        r = step()
        if r is not None:
            r.free()
    torch.cuda.synchronize()

    clocks = {"nvml": NvmlClocks, "nvidia-smi": Clocks}.get(args.clock_sampler, lambda i: None)(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.start()
    times = []
    launches = 0
    last = None
    for _ in range(args.steps):
        if not args.no_flush:
            flush.zero_()  # evict L2 between timed steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if r is not None:  # same allocation pattern as the warm-up: free before the next step
            launches += r.launches
            last = (r.n, r.nl, r.path)
            r.free()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop() if clocks is not None else None
    my_ms = sum(times)
    t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = total_pairs * args.steps / (total_ms / 1e3)
    n_out, nl, path_used = last if last is not None else (0, 1, "none")

    # dominant kernel from live CUDA events (phase timing on the launch stream)
    phase_runs = []
    for _ in range(3):
        flush.zero_()
        r = step(timing=True)
        if r is not None:
            phase_runs.append(r.phases)
            r.free()
    phases = {}
    for pr in phase_runs:
        for k, v in pr.items():
            phases.setdefault(k, []).append(v)
    phases = {k: statistics.median(v) for k, v in phases.items()}
    my_pairs = total_pairs if world == 1 else None

    out = None
    if rank == 0:
        peak, peak_src = hbm_peak()
        # dominant kernel phase: dense numeric pass, radix sort, or bucket reduce
        # (a product can mix bucket and sort batches)
        cands = {k: phases[k] for k in ("numeric", "sort", "reduce", "bucket_reduce") if k in phases}
        kern = max(cands, key=cands.get) if cands else None
        kern_ms = phases.get(kern, float("nan")) if kern else float("nan")
        w_c = 8 if args.coeff == "float" else 8 * nl
        w_in = 8 if A.kind != 2 else 16
        b_alg_step = 32 * total_pairs + (8 + w_c) * n_out + (8 + w_in) * (f.n + g.n)
        kern_pairs = total_pairs / world
        achieved = 32 * kern_pairs / (kern_ms / 1e3) / 1e9 if kern else None
        traffic = None
        prof = ROOT / "profiles" / "numeric_dram_bytes.json"
        if prof.exists():
            try:
                traffic = json.loads(prof.read_text()).get(args.config, {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        kname = {"numeric": f"k_numeric ({path_used} path)",
                 "bucket_reduce": "k_bucket_reduce (bucket path)", "reduce": "k_seg_reduce (sort path)",
                 "sort": "k_rs_onesweep passes (sort path)"}.get(kern, kern)
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "kernel_ms": kern_ms,
                "algorithmic_bytes": "32 B per term product (SURVEY.md 8d: one 16-B pair record "
                                     "written + read); the fused kernel never materialises pairs, "
                                     "so frac > 1 means it moves less than the modelled pipeline",
                "step_frac": b_alg_step / (ms_per_step / 1e3) / 1e9 / (peak * world),
                "phases_ms": phases}
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "int64" if args.coeff == "int" else "f64",
               "data": "synthetic (closed-form Fateman/Monagan-Pearce operands)",
               "config": {"workload": workload_name(args, f, g), "term_products": total_pairs,
                          "result_terms": n_out, "path": path_used, "result_limbs": nl,
                          "arithmetic": ("exact integers: int64 operands, 128-bit products, "
                                         "accumulators proven wide enough (Fateman n=30: 136-bit)")
                          if args.coeff == "int" else "f64",
                          "parallelism": f"partition_by_ops x{world}" if world > 1 else "1 GPU",
                          "gather": {"peer": "peer copies of disjoint slices (CUDA IPC, NVLink)",
                                     "collective": "all-gather of disjoint slices",
                                     "none": "none (1 GPU)"}[gather_kind],
                          "l2": f"flushed ({args.flush_mib} MiB write) between timed steps",
                          "plan_ms": plan_ms, "step_ms": [round(x, 3) for x in times]},
               "roofline": roof, "gpu_launches": launches, "clocks": ck}

    # e2e through the C ABI with pinned host buffers (N=1 only)
    if world == 1 and not args.no_e2e:
        pa_e = torch.from_numpy(A.exps.view(np.int64)).pin_memory()
        pa_c = torch.from_numpy(np.ascontiguousarray(A.coef).view(np.int64).reshape(-1)).pin_memory()
        pb_e = torch.from_numpy(B.exps.view(np.int64)).pin_memory()
        pb_c = torch.from_numpy(np.ascontiguousarray(B.coef).view(np.int64).reshape(-1)).pin_memory()
        h2d = (pa_e.numel() + pa_c.numel() + pb_e.numel() + pb_c.numel()) * 8
        e2e_t = []
        d2h = 0
        for k in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            res = mul_host_pinned(pa_e.data_ptr(), pa_c.data_ptr(), pb_e.data_ptr(), pb_c.data_ptr(),
                                  A.n, B.n, A.kind, f.layout, path=args.path, device=local,
                                  stream=sptr)
            t2 = time.perf_counter()
            d2h = int(res.n) * 8 * (1 + (int(res.acc_limbs) or 1))
            _native.load().pgpu_free_result(__import__("ctypes").byref(res))
            if k >= args.warmup:
                e2e_t.append(t2 - t1)
        if out is not None:
            out["e2e"] = {"value": total_pairs * len(e2e_t) / sum(e2e_t), "unit": UNIT,
                          "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                          "ms_per_step": 1e3 * sum(e2e_t) / len(e2e_t)}
    if args.verify:
        out_v = verify_product(args, f, step, gathered, world, rank)
        if out is not None:
            out["verified"] = out_v
    if out is not None and world == 1 and not args.no_cpu_baseline:
        v, desc, pairs, dt = cpu_sample(f, g, 15.0, cpu_threads())
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                               "sample": desc, "seconds": dt}
    if out is not None:
        print(json.dumps(out), flush=True)
    if peer[0] is not None:
        peer[0].release()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
