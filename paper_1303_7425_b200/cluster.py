"""Multi-GPU product: paper Alg. 2 over torch.distributed (one process per GPU).

The reference simulates N nodes with threads and queues (cluster.py:287-379):
broadcast operands and bounds, compute O_k in `_block` slices, gather them,
cut the intervals into N contiguous ranges of near-equal work
(`partition_by_ops`, cluster.py:261-280), let every node compute its range,
gather the disjoint results.  Here a "node" is a GPU rank:

  1. every rank derives the same bounds (`select_grid`, deterministic);
  2. rank r counts O_k for its `_block` of intervals on its GPU
     (pgpu_count_below) and the counts are all-gathered;
  3. `partition_by_ops` gives each rank a contiguous packed-exponent range
     [S_l1, S_l2); the GPU forms only the products inside it;
  4. the disjoint, already ordered slices are all-gathered into rank order
     (NCCL over NVLink for device tensors; gloo in the CPU tests).  No
     reduction: equal exponents never straddle a bound (split.py:5-9).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import SENTINEL, check_compatible, check_product_fits
from .split import GridParams, select_grid


@dataclass(frozen=True)
class ClusterPlan:
    n_nodes: int
    ranges: tuple
    op_counts: tuple

    def loads(self) -> tuple:
        return tuple(sum(self.op_counts[lo:hi]) for lo, hi in self.ranges)


def partition_by_ops(op_counts, n_nodes: int) -> ClusterPlan:
    """Greedy cumulative cut (reference cluster.py:261-280): range r ends at
    the first prefix whose sum reaches (r+1)/N of the total; each range's load
    exceeds total/N by at most max(op_counts)."""
    if n_nodes < 1:
        raise ValueError(f"need at least one node, got {n_nodes}")
    counts = [int(x) for x in op_counts]
    total = sum(counts)
    cuts = [0]
    run = 0
    k = 0
    for r in range(1, n_nodes):
        while run * n_nodes < r * total:
            run += counts[k]
            k += 1
        cuts.append(k)
    cuts.append(len(counts))
    return ClusterPlan(n_nodes, tuple(zip(cuts[:-1], cuts[1:])), tuple(counts))


def block(n_items: int, n_nodes: int, rank: int) -> tuple:
    """Rank's slice of the interval list for the O_k computation (cluster.py:283-284)."""
    return rank * n_items // n_nodes, (rank + 1) * n_items // n_nodes


def rank_range(bounds, plan: ClusterPlan, rank: int) -> tuple:
    """Packed [lo, hi) of a rank's interval range."""
    l1, l2 = plan.ranges[rank]
    lo = bounds[l1] if l1 < len(bounds) else SENTINEL
    hi = bounds[l2] if l2 < len(bounds) else SENTINEL
    if l1 == l2:
        lo = hi = bounds[l1]
    if l1 == 0:
        lo = 0
    return lo, hi


def _allgather_obj(obj, group):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def plan_for_ranks(a, b, l: int, world: int, rank: int, count_fn, group=None):
    """Bounds + partition, with the O_k of each rank's block all-gathered."""
    bounds = select_grid(a, b, GridParams(l)).bounds
    n_int = len(bounds) - 1
    lo_b, hi_b = block(n_int, world, rank)
    if hi_b > lo_b:
        cum = count_fn(a, b, bounds[lo_b:hi_b + 1])
        mine = [int(cum[k + 1] - cum[k]) for k in range(hi_b - lo_b)]
    else:
        mine = []
    if world > 1:
        parts = _allgather_obj((lo_b, mine), group)
    else:
        parts = [(lo_b, mine)]
    op_counts = [0] * n_int
    for start, cnts in parts:
        op_counts[start:start + len(cnts)] = cnts
    return bounds, partition_by_ops(op_counts, world)


@dataclass
class RankPlan:
    """Paper Alg. 2 for one operand pair, planned once (it depends only on the
    operands' supports, like an FFT plan): the bounds, the partition, every
    rank's packed range, and each range's pair count once known (the library
    reports it with the first product; later products pass it back as
    `range_pairs` and skip the device count)."""
    bounds: list
    plan: ClusterPlan
    ranges: list
    pairs: list

    @property
    def n(self) -> int:
        return self.plan.n_nodes

    def range_of(self, rank: int) -> tuple:
        return self.ranges[rank]


def make_plan(a, b, l: int, world: int, rank: int, count_fn, group=None) -> RankPlan:
    """Each rank counts O_k for its block of intervals; counts all-gathered."""
    bounds, plan = plan_for_ranks(a, b, l, world, rank, count_fn, group)
    return RankPlan(bounds, plan, [rank_range(bounds, plan, r) for r in range(world)], [0] * world)


def rebalance(plan: RankPlan, times) -> RankPlan:
    """Re-cut the intervals by measured cost: partition_by_ops (the reference's
    greedy cumulative cut, cluster.py:261-280) applied to a cost density in
    which interval k of rank r weighs O_k * t_r / P_r (t_r the rank's measured
    product time, P_r its pair count).  Pair counts alone do not balance the
    device work: a range of low-degree terms has short row runs and more row
    visits per pair."""
    op = plan.plan.op_counts
    w = [0.0] * len(op)
    for r, (l1, l2) in enumerate(plan.plan.ranges):
        pr = sum(op[l1:l2])
        if pr == 0:
            continue
        for k in range(l1, l2):
            w[k] = op[k] * float(times[r]) / pr
    tot = sum(w)
    if tot <= 0:
        return plan
    iw = [int(round(x * (1e12 / tot))) for x in w]
    cut = partition_by_ops(iw, plan.n)
    new = ClusterPlan(plan.n, cut.ranges, plan.plan.op_counts)
    return RankPlan(plan.bounds, new, [rank_range(plan.bounds, new, r) for r in range(plan.n)], [0] * plan.n)


def plan_all_ranks(a, b, l: int, n: int, count_fn) -> RankPlan:
    """The N-rank plan computed by one process (every block's O_k on this
    GPU): the virtual-rank mode, where one GPU runs the N range products one
    after another (partition parity at N = 8 on a single device)."""
    bounds = select_grid(a, b, GridParams(l)).bounds
    cum = count_fn(a, b, bounds)
    op_counts = [int(cum[k + 1] - cum[k]) for k in range(len(bounds) - 1)]
    plan = partition_by_ops(op_counts, n)
    return RankPlan(bounds, plan, [rank_range(bounds, plan, r) for r in range(n)], [0] * n)


def gather_slices(exps, coef, group=None, device=None):
    """All-gather disjoint ordered slices (torch tensors) into rank order.

    exps: (n,) int64 view of the u64 exponents; coef: (n, w) int64 view of the
    coefficient words.  Returns the concatenation on every rank.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) != "nccl":  # gloo collectives run on host tensors
        exps, coef = exps.cpu(), coef.cpu()
    n = torch.tensor([exps.shape[0]], dtype=torch.int64, device=exps.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    counts = [int(x.item()) for x in ns]
    m = max(counts) if counts else 0
    w = coef.shape[1]
    if m == 0:
        return exps[:0], coef[:0]
    pe = torch.zeros(m, dtype=torch.int64, device=exps.device)
    pc = torch.zeros((m, w), dtype=torch.int64, device=exps.device)
    pe[:exps.shape[0]] = exps
    pc[:exps.shape[0]] = coef
    if dist.get_backend(group) == "nccl":
        ge = torch.empty(world * m, dtype=torch.int64, device=exps.device)
        gc = torch.empty((world * m, w), dtype=torch.int64, device=exps.device)
        dist.all_gather_into_tensor(ge, pe, group=group)
        dist.all_gather_into_tensor(gc, pc, group=group)
    else:  # gloo (CPU tests, single-GPU rank emulation): list all-gather on host tensors
        pe, pc = pe.cpu(), pc.cpu()
        le = [torch.empty_like(pe) for _ in range(world)]
        lc = [torch.empty_like(pc) for _ in range(world)]
        dist.all_gather(le, pe, group=group)
        dist.all_gather(lc, pc, group=group)
        ge, gc = torch.cat(le), torch.cat(lc)
    es = [ge[r * m:r * m + counts[r]] for r in range(world)]
    cs = [gc[r * m:r * m + counts[r]] for r in range(world)]
    return torch.cat(es), torch.cat(cs)


class PeerGather:
    """The final step of paper Alg. 2 as peer copies over NVLink (the north
    star's "peer copies, no reduction collective").  The destination rank(s)
    hold the assembled product in a CUDA-IPC-shareable buffer whose handle the
    other ranks open once; each rank copies its own ordered slice straight
    into the destination buffer at its offset (device to device, through the
    peer mapping).  dst = r: only rank r assembles (N-1 copies, the
    reference's gather to node 0, cluster.py:311-317); dst = None: every rank
    does (an all-gather).

    Per step under NCCL the synchronisation is stream-ordered: the term counts
    are one all-gather of an int64, and completion is an all-reduce of one
    word enqueued after the copies (each rank's copies precede it on its
    stream), so no host barrier and no pickled object exchange.  Buffers and
    peer mappings are reused while the assembled size stays the same."""

    def __init__(self, group=None, device: int = 0, dst: int | None = None):
        import torch
        import torch.distributed as dist
        from . import _native as N
        self.N, self.lib = N, N.load()
        self.group, self.device, self.dst_rank = group, device, dst
        self.nccl = dist.get_backend(group) == "nccl"
        self.shape = None
        self.bufs, self.dst = [], []
        dev = torch.device("cuda", device)
        self.cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        self.cnts = torch.zeros(dist.get_world_size(group), dtype=torch.int64, device=dev)
        self.tick = torch.zeros(1, dtype=torch.int32, device=dev)

    def _check(self, st):
        if st != self.N.PGPU_OK:
            raise self.N.NativeError(self.N.last_error())

    def _dests(self, world):
        return list(range(world)) if self.dst_rank is None else [self.dst_rank]

    def _setup(self, total: int, w: int):
        import ctypes as C
        import torch.distributed as dist
        self.release()
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        handles = None
        if rank in self._dests(world):
            handles = []
            for nbytes in (total * 8, total * w * 8):
                ptr, h = C.c_void_p(), C.create_string_buffer(self.N.IPC_HANDLE_BYTES)
                self._check(self.lib.pgpu_ipc_alloc(nbytes, self.device, C.byref(ptr), h))
                self.bufs.append(ptr.value)
                handles.append(h.raw)
        peers = _allgather_obj(handles, self.group)  # once per assembled shape
        self.dst = []
        for r in self._dests(world):
            if r == rank:
                self.dst.append((self.bufs[0], self.bufs[1], False))
                continue
            opened = []
            for h in peers[r]:
                ptr = C.c_void_p()
                self._check(self.lib.pgpu_ipc_open(h, self.device, C.byref(ptr)))
                opened.append(ptr.value)
            self.dst.append((opened[0], opened[1], True))
        self.shape = (total, w)

    def counts(self, n: int) -> list:
        import torch.distributed as dist
        if self.nccl:
            self.cnt.fill_(n)
            dist.all_gather_into_tensor(self.cnts, self.cnt, group=self.group)
            return [int(x) for x in self.cnts.tolist()]
        return [int(x) for x in _allgather_obj(n, self.group)]

    def gather(self, exps, coef, stream=None):
        """(exps int64[total], coef int64[total, w]) views of the assembled
        product on a destination rank; None on the others."""
        import torch
        import torch.distributed as dist
        from .device import _CudaArray
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        n, w = int(exps.shape[0]), int(coef.shape[1])
        counts = self.counts(n)
        off = sum(counts[:rank])
        total = sum(counts)
        if self.shape != (total, w):
            self._setup(total, w)
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        for de, dc, _ in self.dst:
            self._check(self.lib.pgpu_copy(de + off * 8, exps.data_ptr(), n * 8, self.device, st))
            self._check(self.lib.pgpu_copy(dc + off * w * 8, coef.data_ptr(), n * w * 8, self.device, st))
        if self.nccl:
            dist.all_reduce(self.tick, group=self.group)  # stream-ordered: all slices in place
        else:  # gloo (rank emulation): host-side completion
            self._check(self.lib.pgpu_stream_sync(self.device, st))
            dist.barrier(self.group)
        if rank not in self._dests(world):
            return None
        dev = torch.device("cuda", self.device)
        if total == 0:
            return torch.zeros(0, dtype=torch.int64, device=dev), torch.zeros((0, w), dtype=torch.int64, device=dev)
        return (torch.as_tensor(_CudaArray(self.bufs[0], (total,), "<i8"), device=dev),
                torch.as_tensor(_CudaArray(self.bufs[1], (total, w), "<i8"), device=dev))

    def release(self):
        """Unmap the peers' buffers and free ours (collective: call on every rank)."""
        import torch.distributed as dist
        if self.shape is None:
            return
        dist.barrier(self.group)  # nobody still writes into our buffers
        for de, dc, opened in self.dst:
            if opened:
                self.lib.pgpu_ipc_close(de)
                self.lib.pgpu_ipc_close(dc)
        dist.barrier(self.group)  # peers unmapped before the memory goes away
        for ptr in self.bufs:
            self.lib.pgpu_ipc_free(ptr)
        self.bufs, self.dst, self.shape = [], [], None


def gpu_mul(a, b, cfg=None, *, group=None, local_fn=None, count_fn=None):
    """Distributed product; every rank returns the full Polynomial.

    `local_fn(a, b, lo, hi) -> RawProduct` and `count_fn(a, b, bounds)` default
    to the CUDA library (parmul.native_mul / count_below); the CPU tests inject
    oracle versions to exercise the partition and gather logic over gloo.
    """
    import torch
    import torch.distributed as dist
    from . import parmul
    cfg = parmul.MulConfig.of(cfg)
    check_compatible(a, b)
    cls = type(a)
    if a.is_zero or b.is_zero:
        return cls.zero(a.layout, a.ctype)
    check_product_fits(a, b)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if count_fn is None:
        def count_fn(x, y, bnd):
            return parmul.count_below(x, y, bnd, device=cfg.device)
    device_path = local_fn is None and world > 1
    if local_fn is None:
        def local_fn(x, y, lo, hi):
            return parmul.native_mul(parmul.Operand.from_poly(x), parmul.Operand.from_poly(y),
                                     x.layout, lo=lo, hi=hi, path=cfg.path,
                                     float_ordered=cfg.ordered, device=cfg.device)
    bounds, plan = plan_for_ranks(a, b, cfg.l, world, rank, count_fn, group)
    lo, hi = rank_range(bounds, plan, rank)
    if device_path:
        return _gpu_range_and_peer_gather(a, b, cfg, lo, hi, group)
    if lo < hi:
        raw = local_fn(a, b, lo, hi)
    else:
        raw = None
    if world == 1:
        if raw is None:
            return cls.zero(a.layout, a.ctype)
        return parmul.to_poly(cls, a.layout, a.ctype, raw)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    # coefficient words: f64 bit patterns or u64 limbs; widths agree across ranks
    if raw is None:
        e = np.zeros(0, np.uint64)
        wd = 1
        cw = np.zeros((0, 1), np.uint64)
        kind = None
    else:
        e = raw.exps
        cw = raw.coef.view(np.uint64).reshape(raw.exps.shape[0], -1)
        wd = cw.shape[1]
        kind = (raw.kind, raw.nl)
    kinds = _allgather_obj((kind, wd), group)
    wd = max(k[1] for k in kinds)
    kind = next((k[0] for k in kinds if k[0] is not None), None)
    if cw.shape[1] < wd:  # sign-extend narrower limb sets
        ext = np.empty((cw.shape[0], wd), np.uint64)
        ext[:, :cw.shape[1]] = cw
        sign = (cw[:, -1].view(np.int64) >> 63).view(np.uint64) if cw.shape[0] else np.zeros(0, np.uint64)
        for k in range(cw.shape[1], wd):
            ext[:, k] = sign
        cw = ext
    te = torch.from_numpy(e.view(np.int64).copy()).to(dev)
    tc = torch.from_numpy(cw.view(np.int64).copy()).to(dev)
    ge, gc = gather_slices(te, tc, group)
    exps = ge.cpu().numpy().view(np.uint64)
    words = gc.cpu().numpy().view(np.uint64)
    if kind is None:
        return cls.zero(a.layout, a.ctype)
    nkind, nl = kind
    if a.ctype is float:
        coef = words.reshape(-1).view(np.float64)
    else:
        coef = words
        nl = wd
    raw_all = parmul.RawProduct(exps, coef, nkind, nl, 0, "", 0, 0, {})
    return parmul.to_poly(cls, a.layout, a.ctype, raw_all)


def _gpu_range_and_peer_gather(a, b, cfg, lo, hi, group):
    """One rank's range product left on its GPU, then the peer-copy gather
    (PeerGather) and a single device-to-host copy of the assembled product."""
    import numpy as np
    import torch
    from . import parmul
    from .device import DeviceOperand, mul_on_device
    cls = type(a)
    dev = torch.device("cuda", cfg.device)
    res = None
    if lo < hi:
        dA = DeviceOperand(parmul.Operand.from_poly(a), dev)
        dB = DeviceOperand(parmul.Operand.from_poly(b), dev)
        res = mul_on_device(dA, dB, a.layout, lo=lo, hi=hi, path=cfg.path,
                            float_ordered=cfg.ordered, device=cfg.device)
    try:
        if res is not None and res.n:
            e, c = res.tensors()
            c = c.view(torch.int64).reshape(e.shape[0], -1)
            kind = (res.kind, res.nl)
        else:
            e = torch.zeros(0, dtype=torch.int64, device=dev)
            c = torch.zeros((0, 1), dtype=torch.int64, device=dev)
            kind = None
        kinds = _allgather_obj((kind, int(c.shape[1])), group)
        wd = max(k[1] for k in kinds)
        kind = next((k[0] for k in kinds if k[0] is not None), None)
        if c.shape[1] < wd:  # sign-extend narrower limb sets (exact ints)
            sign = (c[:, -1:] >> 63).expand(-1, wd - c.shape[1])
            c = torch.cat([c, sign], dim=1)
        pg = PeerGather(group, cfg.device)
        try:
            ge, gc = pg.gather(e.contiguous(), c.contiguous())
            exps = ge.cpu().numpy().view(np.uint64)
            words = gc.cpu().numpy().view(np.uint64)
        finally:
            pg.release()
    finally:
        if res is not None:
            res.free()
    if kind is None:
        return cls.zero(a.layout, a.ctype)
    nkind, nl = kind
    if a.ctype is float:
        coef = words.reshape(-1).view(np.float64)
    else:
        coef, nl = words, wd
    return parmul.to_poly(cls, a.layout, a.ctype, parmul.RawProduct(exps, coef, nkind, nl, 0, "", 0, 0, {}))
