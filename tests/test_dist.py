"""World-size-2 gloo run of the multi-GPU plan (paper Alg. 2): bounds,
O_k computed per rank block and all-gathered, partition_by_ops ranges, and
the rank-ordered all-gather of disjoint slices.  The per-rank product and
op counts are injected from the oracle (no GPU here); on a GPU box the same
code calls the CUDA library."""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_local(a, b, lo, hi):
    from oracle import oracle as O
    from paper_1303_7425_b200.parmul import RawProduct, int_coeff_array
    exps, co = O.mul_raw(a, b, bounds=[lo, hi] if hi != (1 << 64) - 1 else [lo, hi],
                         k_range=(0, 1))
    # oracle with a 2-bound split forms the products in [lo, hi)
    if a.ctype is float:
        coef = np.asarray(co, dtype=np.float64)
        return RawProduct(exps, coef, 0, 1, 0, "oracle", 0, 0, {})
    limbs = np.zeros((len(co), 3), dtype=np.uint64)
    m = (1 << 64) - 1
    for k, c in enumerate(co):
        limbs[k] = [c & m, (c >> 64) & m, (c >> 128) & m]
    return RawProduct(exps, limbs, 1, 3, 0, "oracle", 0, 0, {})


def _oracle_count(a, b, bounds):
    # cum[k] = #pairs below bounds[k]
    ae = np.asarray(a.exps, dtype=np.uint64)
    be = np.asarray(b.exps, dtype=np.uint64)
    sums = (ae[:, None] + be[None, :]).ravel()
    return [int(np.count_nonzero(sums < np.uint64(x))) for x in bounds]


def _worker(rank, world, port, ctype_name, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1303_7425_b200 import benchpolys, gpu_mul, MulConfig
        ct = float if ctype_name == "float" else int
        f, g = benchpolys.fateman(5, ct)
        p = gpu_mul(f, g, MulConfig(l=8), local_fn=_oracle_local, count_fn=_oracle_count)
        q.put((rank, p.exps, p.coeffs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ctype_name", ["int", "float"])
def test_two_rank_partition_and_gather(ctype_name):
    from oracle import oracle as O
    from paper_1303_7425_b200 import benchpolys
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ctype_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ct = float if ctype_name == "float" else int
    f, g = benchpolys.fateman(5, ct)
    want = O.mul(f, g)
    for rank, exps, coeffs in outs:
        assert exps == want.exps
        assert coeffs == want.coeffs
