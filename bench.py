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
    ap.add_argument("--rebalance", type=int, default=2,
                    help="N>1: rounds of cost rebalancing of the partition during warm-up")
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
    """Synthetic operands of the config: exact ints in closed form (identical
    to the reference's poly_from_expr output); floats as the reference builds
    them, by repeated squaring in float (the GPU powering in its order)."""
    from paper_1303_7425_b200 import benchpolys
    if args.coeff == "float" and _gpu_present():
        return benchpolys.reference_float_operands(args.config)
    ct = float if args.coeff == "float" else int
    return benchpolys.CONFIGS[args.config](ct)


def _gpu_present() -> bool:
    try:
        from paper_1303_7425_b200 import _native
        return _native.load().pgpu_device_count() > 0
    except Exception:
        return False


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


def python_reference_sample(f, g, threads, frac_den=64):
    """The reference's own Python path (baseline/_ref, installed from
    /root/reference by pip) on a contiguous 1/frac_den slice of its
    select_grid(l=64) intervals: compute_intervals with its fork pool of
    `threads` workers (parmul.py:64-88).  Returns a dict, or None when the
    install is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "polymul").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from polymul import core as rcore
        from polymul import parmul as rparmul
        from polymul import split as rsplit
    except Exception as exc:  # pragma: no cover - install broken
        return {"unavailable": f"import failed: {exc}"}
    lay = rcore.default_layout(tuple(f.layout.vars.names), f.layout.order)
    ra = rcore.Polynomial._from_sorted(lay, list(f.exps), list(f.coeffs), f.ctype)
    rb = rcore.Polynomial._from_sorted(lay, list(g.exps), list(g.coeffs), g.ctype)
    bounds = rsplit.select_grid(ra, rb, rsplit.GridParams(64)).bounds
    n_int = len(bounds) - 1
    width = max(1, n_int // frac_den)
    start = (n_int - width) // 2
    pairs = int(sum(rparmul.interval_op_counts(ra, rb, bounds, start, start + width)))
    t0 = time.perf_counter()
    rparmul.compute_intervals(ra, rb, bounds, start, start + width, "heap", threads)
    dt = time.perf_counter() - t0
    return {"value": pairs / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"intervals [{start}, {start + width}) of {n_int} select_grid(l=64) intervals "
                      f"({pairs} of {f.n * g.n} term products), reference polymul.parmul."
                      f"compute_intervals (heap merger, fork pool of {threads})",
            "seconds": dt}


def run_reference(args):
    """The reference's CPU algorithm on the box's host cores: the oracle's C
    restatement of select_grid -> find_edge -> heap_merge over EVERY interval
    of the product each timed step (the whole workload, all host threads),
    plus one timing of the reference's own Python path on a 1/64 slice."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    from oracle import oracle as O
    f, g = operands(args)
    threads = cpu_threads()
    bounds = O.select_grid(f, g, 64)
    P = f.n * g.n
    full = os.environ.get("REF_SAMPLE_STRIDE") is None
    stride = 1 if full else int(os.environ["REF_SAMPLE_STRIDE"])
    pairs = P if stride == 1 else O.sample_pairs(f, g, bounds, stride)
    # warm-up steps are untimed: a 1/64 sample each (the whole product takes
    # ~10 s per step on 16 threads)
    for _ in range(args.warmup):
        O.mul_raw(f, g, threads=threads, bounds=bounds, stride=64)
    tt = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.mul_raw(f, g, threads=threads, bounds=bounds, stride=stride)
        tt.append(time.perf_counter() - t0)
    value = pairs * len(tt) / sum(tt)
    desc = (f"every interval of {len(bounds) - 1} select_grid(l=64) intervals ({P} term products: the whole "
            f"product), C heap_merge port, {threads} threads" if stride == 1 else
            f"every {stride}th of {len(bounds) - 1} intervals ({pairs} of {P} term products), C heap_merge "
            f"port, {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(tt) / max(1, len(tt)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64" if args.coeff == "int" else "f64", "data": "synthetic (closed form)",
            "impl": "reference",
            "config": {"workload": workload_name(args, f, g), "sample": desc, "cpu_model": cpu_model()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": desc, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not os.environ.get("NO_PY_REFERENCE"):
        try:
            line["python_reference"] = python_reference_sample(f, g, threads)
        except Exception as exc:  # reported, never fatal for the CPU arm
            line["python_reference"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        pr = line["python_reference"]
        if pr and "value" in pr:
            line["python_reference"]["port_speedup"] = value / pr["value"]
    print(json.dumps(line), flush=True)
    return 0


def verify_product(args, f, step, gathered, world, rank):
    """sha256 of the reference text format of the (assembled) product vs the
    reference's recorded digest (tests/golden/digests.json); rank 0 only."""
    import numpy as np
    from paper_1303_7425_b200 import io
    from paper_1303_7425_b200.core import Polynomial
    from paper_1303_7425_b200.parmul import limbs_to_ints
    want = json.loads((ROOT / "tests" / "golden" / "digests.json").read_text())["products"]
    key = f"{args.config}/{args.coeff}"
    r = step()
    exps = words = None
    if rank == 0:
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
    if rank != 0:
        return None
    if args.coeff == "float":
        co = words.reshape(-1).view(np.float64).tolist()
    else:
        co = limbs_to_ints(words, words.shape[1])
    p = Polynomial._from_sorted(f.layout, exps.tolist(), co, float if args.coeff == "float" else int)
    got = io.poly_digest(p)
    ok = key in want and want[key]["sha256"] == got
    return {"digest": got, "reference_digest": want.get(key, {}).get("sha256"), "ok": ok, "terms": p.n}


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1.  With fewer devices than
    ranks the ranks are emulated on the available devices over gloo (a
    correctness run: the line says so, and its times are not a scaling
    measurement)."""
    from paper_1303_7425_b200 import _native
    ndev = _native.load().pgpu_device_count()
    argv = list(sys.argv[1:])
    if ndev < args.gpus and not args.emulate_ranks:
        print(f"[bench] {args.gpus} ranks requested, {ndev} CUDA device(s) visible: emulating the ranks "
              "over gloo (correctness only)", file=sys.stderr, flush=True)
        argv.append("--emulate-ranks")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1303_7425_b200 import _native
    from paper_1303_7425_b200.cluster import PeerGather, gather_slices, make_plan
    from paper_1303_7425_b200.core import SENTINEL
    from paper_1303_7425_b200.device import (DeviceOperand, PinnedOperand, mul_host_pinned,
                                             mul_on_device)
    from paper_1303_7425_b200.parmul import Operand, count_below

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    ndev = _native.load().pgpu_device_count()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.emulate_ranks:
        local = local % max(1, ndev)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.emulate_ranks:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    f, g = operands(args)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    dA, dB = DeviceOperand(A, dev), DeviceOperand(B, dev)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # partition (paper Alg. 2): planned once per operand pair, timed separately
    t0 = time.perf_counter()
    lo, hi = 0, SENTINEL
    plan = None
    if world > 1:
        plan = make_plan(f, g, 64, world, rank, lambda x, y, b: count_below(x, y, b, device=local))
        lo, hi = plan.range_of(rank)
    plan_ms = 1e3 * (time.perf_counter() - t0)
    my_pairs = [0]  # this range's pair count, reported by the first product (the plan's cache)

    total_pairs = f.n * g.n
    gathered = [None]
    gather_kind = "none"
    peer = None
    if world > 1:
        gather_kind = args.gather
        if args.gather == "peer":
            peer = PeerGather(device=local, dst=0)

    def range_product(Ain, Bin, timing=False, inputs_on_device=True):
        if lo >= hi:
            return None
        r = mul_on_device(Ain, Bin, f.layout, lo=lo, hi=hi, path=args.path, device=local, stream=sptr,
                          timing=timing, range_pairs=my_pairs[0], inputs_on_device=inputs_on_device)
        my_pairs[0] = r.pairs
        return r

    def gather(res):
        if res is not None:
            e, c = res.tensors()
            c = c.view(torch.int64).reshape(e.shape[0], -1)
        else:
            e = torch.zeros(0, dtype=torch.int64, device=dev)
            c = torch.zeros((0, 3 if args.coeff == "int" else 1), dtype=torch.int64, device=dev)
        if peer is not None:
            gathered[0] = peer.gather(e, c, stream=sptr)
        else:
            gathered[0] = gather_slices(e, c)

    def step(timing=False, ev=None):
        res = range_product(dA, dB, timing=timing)
        if world > 1:
            if ev is not None:
                ev.record(stream)
            gather(res)
        return res

    flush = torch.empty(args.flush_mib * (1 << 20) // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        r = step()
        if r is not None:
            r.free()
    torch.cuda.synchronize()
    rebalanced = 0
    if world > 1 and args.rebalance > 0:
        # cost balancing (part of the plan): every rank times its own range
        # product, the times are all-gathered, and the intervals are re-cut
        # by partition_by_ops on the measured cost density (cluster.rebalance)
        from paper_1303_7425_b200.cluster import rebalance
        for _ in range(args.rebalance):
            ts = []
            for _ in range(3):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = range_product(dA, dB)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
                if r is not None:
                    r.free()
            mine = torch.tensor([statistics.median(ts)], dtype=torch.float64)
            allt = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            if args.emulate_ranks:
                dist.all_gather(allt, mine)
            else:
                allt = [x.to(dev) for x in allt]
                dist.all_gather(allt, mine.to(dev))
            plan = rebalance(plan, [float(x.item()) for x in allt])
            lo, hi = plan.range_of(rank)
            my_pairs[0] = 0
            rebalanced += 1
        for _ in range(2):  # warm the new ranges (pair counts, workspace)
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
    times, prod_ms = [], []
    launches = 0
    last = None
    for _ in range(args.steps):
        if not args.no_flush:
            flush.zero_()  # evict L2 between timed steps
        e0 = torch.cuda.Event(enable_timing=True)
        em = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = step(ev=em)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if world > 1:
            prod_ms.append(e0.elapsed_time(em))
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
        if args.emulate_ranks:
            t = t.cpu()
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
    multi = None
    if world > 1:
        # per step: range product vs gather + synchronisation (max over ranks)
        mine = [statistics.median(prod_ms), statistics.median([a - b for a, b in zip(times, prod_ms)])]
        tt = torch.tensor(mine, dtype=torch.float64, device=dev)
        if args.emulate_ranks:
            tt = tt.cpu()
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nterms = torch.tensor([float(n_out)], dtype=torch.float64, device=dev)
        nterms = nterms.cpu() if args.emulate_ranks else nterms
        dist.all_reduce(nterms)
        multi = {"product_ms": float(tt[0]), "gather_ms": float(tt[1]),
                 "non_product_ms": ms_per_step - float(tt[0]), "terms": int(nterms.item())}
        phases["gather"] = float(tt[1])

    out = None
    if rank == 0:
        peak, peak_src = hbm_peak()
        # dominant kernel phase: dense numeric pass, radix sort, or bucket reduce
        # (a product can mix bucket and sort batches)
        cands = {k: phases[k] for k in ("numeric", "sort", "reduce", "bucket_reduce") if k in phases}
        kern = max(cands, key=cands.get) if cands else None
        kern_ms = phases.get(kern, float("nan")) if kern else float("nan")
        n_all = multi["terms"] if multi else n_out
        w_c = 8 if args.coeff == "float" else 8 * nl
        w_in = 8 if A.kind != 2 else 16
        b_alg_step = 32 * total_pairs + (8 + w_c) * n_all + (8 + w_in) * (f.n + g.n)
        kern_pairs = total_pairs / world
        achieved = 32 * kern_pairs / (kern_ms / 1e3) / 1e9 if kern else None
        kfam = {"numeric": "k_numeric", "bucket_reduce": "k_bucket_reduce", "reduce": "k_seg_reduce",
                "sort": "k_rs_"}.get(kern)
        traffic, traffic_src = None, None
        prof = ROOT / "profiles" / "dram_bytes.json"
        if prof.exists() and kfam:  # ncu-measured DRAM bytes of the kernel over one product
            try:
                rec = json.loads(prof.read_text()).get(f"{args.config}/{args.coeff}", {})
                hit = {k: v for k, v in rec.get("kernels", {}).items() if k.startswith(kfam)}
                if hit and world == 1:
                    traffic = sum(v["dram_bytes"] for v in hit.values())
                    traffic_src = rec.get("source")
            except Exception:
                traffic = None
        kname = {"numeric": f"k_numeric ({path_used} path)",
                 "bucket_reduce": "k_bucket_reduce (bucket path)", "reduce": "k_seg_reduce (sort path)",
                 "sort": "radix passes k_rs_count/k_rs_colscan/k_rs_scatter (sort path)"}.get(kern, kern)
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": peak_src, "kernel_ms": kern_ms,
                "algorithmic_bytes": "32 B per term product (SURVEY.md 8d: one 16-B pair record "
                                     "written + read) over the kernel's time; the fused dense kernel "
                                     "never materialises pairs, so frac > 1 means it moves less than "
                                     "the modelled pipeline",
                "step_frac": b_alg_step / (ms_per_step / 1e3) / 1e9 / (peak * world),
                "phases_ms": phases}
        if kern == "numeric":
            # the dense kernel's real limiter is the shared-memory / L1 pipe:
            # per term product a 16-byte accumulator read-modify-write (32 B)
            # plus the 2-byte slot-table lookup, against 128 B/clk per SM
            sm_mhz = (ck or {}).get("sm_mhz") or 1965.0
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            smem_peak = 128.0 * nsm * sm_mhz * 1e6 / 1e9
            smem_ach = 34.0 * kern_pairs / (kern_ms / 1e3) / 1e9
            roof["bound"] = "smem"
            roof["smem"] = {"achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
                            "frac": smem_ach / smem_peak, "bytes_per_pair": 34,
                            "peak_def": f"128 B/clk x {nsm} SMs x {sm_mhz:.0f} MHz (median SM clock "
                                        "under load)",
                            "note": "frac (above) is the SURVEY 8(d) HBM model; the kernel moves "
                                    "~0.3 GB of DRAM per product (traffic) and is bound by the "
                                    "shared-memory/L1 pipe"}
        emulated = bool(args.emulate_ranks and world > 1)
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "int64" if args.coeff == "int" else "f64",
               "data": ("synthetic: closed-form Fateman/Monagan-Pearce operands (exact ints)" if args.coeff == "int" else "synthetic: the reference's float operands (repeated squaring in float, reference order)"),
               "config": {"workload": workload_name(args, f, g), "term_products": total_pairs,
                          "result_terms": n_all, "path": path_used, "result_limbs": nl,
                          "arithmetic": ("exact integers: int64 operands, 128-bit products, "
                                         "accumulators proven wide enough (Fateman n=30: 136-bit)")
                          if args.coeff == "int" else "f64",
                          "parallelism": (f"partition_by_ops x{world}" +
                                          (f", ranks emulated on {max(1, ndev)} device(s) over gloo "
                                           "(correctness run; times are not a scaling measurement)"
                                           if emulated else "")) if world > 1 else "1 GPU",
                          "gather": {"peer": "peer copies of disjoint slices to rank 0 (CUDA IPC, "
                                             "NVLink); counts and completion " +
                                             ("exchanged over gloo" if args.emulate_ranks else
                                              "stream-ordered over NCCL"),
                                     "collective": "all-gather of disjoint slices",
                                     "none": "none (1 GPU)"}[gather_kind],
                          "l2": f"flushed ({args.flush_mib} MiB write) between timed steps",
                          "plan": ("select_grid(l=64) + O_k partition (partition_by_ops), "
                                   f"{rebalanced} round(s) of re-cutting by measured cost, and each range's "
                                   "pair count from the first product: once per operand pair")
                          if world > 1 else "none (1 GPU)",
                          "plan_ms": plan_ms, "step_ms": [round(x, 3) for x in times]},
               "roofline": roof, "gpu_launches": launches, "clocks": ck}
        if multi:
            out["multi_gpu"] = multi
        if emulated:
            out["emulated_ranks"] = True

    # e2e through the public API with host buffers (H2D of the operands and
    # D2H of the assembled product inside the timed region)
    if not args.no_e2e:
        if world == 1:
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
            e2e_s = sum(e2e_t) / len(e2e_t)
        else:
            # each rank: pinned operands in, its range product, peer gather to
            # rank 0; rank 0 copies the assembled product to pinned host memory
            pA, pB = PinnedOperand(A), PinnedOperand(B)
            h2d = pA.bytes + pB.bytes
            host_out = [None]
            e2e_t = []
            d2h = 0
            for k in range(args.warmup + args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                dist.barrier()
                t1 = time.perf_counter()
                r = range_product(pA, pB, inputs_on_device=False)
                gather(r)
                if rank == 0 and gathered[0] is not None:
                    ge, gc = gathered[0]
                    if host_out[0] is None or host_out[0][0].shape != ge.shape or host_out[0][1].shape != gc.shape:
                        host_out[0] = (torch.empty(ge.shape, dtype=ge.dtype, pin_memory=True),
                                       torch.empty(gc.shape, dtype=gc.dtype, pin_memory=True))
                    host_out[0][0].copy_(ge, non_blocking=True)
                    host_out[0][1].copy_(gc, non_blocking=True)
                    d2h = (ge.numel() + gc.numel()) * 8
                torch.cuda.synchronize()
                t2 = time.perf_counter()
                if r is not None:
                    r.free()
                if k >= args.warmup:
                    e2e_t.append(t2 - t1)
            mine = torch.tensor([sum(e2e_t) / len(e2e_t)], dtype=torch.float64, device=dev)
            mine = mine.cpu() if args.emulate_ranks else mine
            dist.all_reduce(mine, op=dist.ReduceOp.MAX)
            e2e_s = float(mine.item())
        if out is not None:
            out["e2e"] = {"value": total_pairs / e2e_s, "unit": UNIT,
                          "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h,
                          "ms_per_step": 1e3 * e2e_s}
        if world == 1 and out is not None:
            # the reference-facing call: Polynomial (Python int/float lists) in,
            # Polynomial out -- marshaling both ways inside the timed region
            from paper_1303_7425_b200 import MulConfig, mul
            cfg = MulConfig(path=args.path, float_ordered=False, device=local)
            api_t = []
            for k in range(2 + min(args.steps, 5)):
                t1 = time.perf_counter()
                p = mul(f, g, cfg)
                t2 = time.perf_counter()
                if k >= 2:
                    api_t.append(t2 - t1)
                del p
            api_s = sum(api_t) / len(api_t)
            out["e2e_api"] = {"value": total_pairs / api_s, "unit": UNIT, "ms_per_step": 1e3 * api_s,
                              "steps": len(api_t),
                              "call": "paper_1303_7425_b200.mul(Polynomial, Polynomial) -> Polynomial: "
                                      "Python int lists marshaled in and out (the reference's parmul.mul "
                                      "signature, parmul.py:91-109)"}
    if args.verify:
        out_v = verify_product(args, f, step, gathered, world, rank)
        if out is not None:
            out["verified"] = out_v
    if out is not None and not args.no_cpu_baseline:
        v, desc, pairs, dt = cpu_sample(f, g, 15.0, cpu_threads())
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                               "sample": desc, "seconds": dt, "cpu_model": cpu_model()}
    if out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        if peer is not None:
            peer.release()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


if __name__ == "__main__":
    sys.exit(main())
