"""Paper Alg. 2 at N = 8 on one GPU ("virtual ranks"): the 8 partition_by_ops
ranges (reference cluster.py:261-319) of a product are computed one after
another on cuda:0, exactly as 8 ranks would compute them, and the
concatenation in rank order must be the product:

  * Fateman n=30: the concatenation carries the reference's digest;
  * MP n=25 (2.03e10 term products): 312,855,140 terms, the
    69 reference sampled-interval digests (each interval lies inside one
    rank's range), and the modular evaluation checksum of the whole product.
"""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from conftest import digests, product_digest
from paper_1303_7425_b200 import benchpolys, io
from paper_1303_7425_b200.cluster import plan_all_ranks
from paper_1303_7425_b200.core import Polynomial
from paper_1303_7425_b200.parmul import Operand, count_below, limbs_to_ints, native_mul

pytestmark = pytest.mark.gpu
N = 8


def _plan(f, g):
    plan = plan_all_ranks(f, g, 64, N, lambda a, b, bnd: count_below(a, b, bnd))
    loads = plan.plan.loads()
    assert len(plan.ranges) == N and sum(loads) == f.n * g.n
    assert max(loads) <= sum(loads) / N + max(plan.plan.op_counts)  # cluster.py:261-280 bound
    # ranges tile the key space in order
    for (lo0, hi0), (lo1, hi1) in zip(plan.ranges, plan.ranges[1:]):
        assert hi0 == lo1
    return plan


def test_fateman30_eight_ranges_concatenate_to_the_reference_product():
    f, g = benchpolys.fateman(30)
    plan = _plan(f, g)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    exps, coefs, pairs = [], [], 0
    for lo, hi in plan.ranges:
        raw = native_mul(A, B, f.layout, lo=lo, hi=hi)
        pairs += raw.pairs
        exps.extend(raw.exps.tolist())
        coefs.extend(limbs_to_ints(raw.coef, raw.nl))
    assert pairs == f.n * g.n
    p = Polynomial._from_sorted(f.layout, exps, coefs, int)
    want = digests()["products"]["fateman30/int"]
    assert p.n == want["n"] and io.poly_digest(p) == want["sha256"]


def test_mp25_eight_ranges_count_sampled_intervals_and_checksum():
    import torch
    from test_gpu_checksum import P, eval_device, eval_host
    from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
    d = digests()["mp25_intervals"]
    f, g = benchpolys.monagan_pearce(25)
    plan = _plan(f, g)
    bounds = plan.bounds
    assert len(bounds) == d["n_s"]
    dev = torch.device("cuda", 0)
    dA, dB = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
    rng = random.Random(0x25)
    pts = [[rng.randrange(2, P - 1) for _ in range(f.layout.vars.m)] for _ in range(2)]
    sums = [0, 0]
    rows = {r["k"]: r for r in d["rows"]}
    ks = list(range(0, 4289, 64)) + [4322]
    per_k = {}
    total_terms = 0
    for r, (l1, l2) in enumerate(plan.plan.ranges):
        lo, hi = plan.ranges[r]
        if lo >= hi:
            continue
        res = mul_on_device(dA, dB, f.layout, lo=lo, hi=hi)
        try:
            total_terms += res.n
            for t, pt in enumerate(pts):
                sums[t] = (sums[t] + eval_device(res, f.layout, pt)) % P
            e, c = res.tensors()
            eu = e.cpu().numpy().view(np.uint64)
            for k in ks:
                if not (l1 <= k < l2):
                    continue
                a = int(np.searchsorted(eu, np.uint64(bounds[k]), "left")) if k else 0
                b = int(np.searchsorted(eu, np.uint64(bounds[k + 1]), "left")) if k + 1 < len(bounds) - 1 \
                    else eu.shape[0]
                words = c[a:b].cpu().numpy().view(np.uint64).reshape(b - a, -1)
                per_k[k] = product_digest(eu[a:b].tolist(), limbs_to_ints(words, words.shape[1]))
                if k in rows:
                    assert b - a == rows[k]["terms"]
        finally:
            res.free()
            torch.cuda.empty_cache()
    assert total_terms == 312_855_140
    for k, r in rows.items():
        assert per_k[k] == r["sha256"], f"interval {k}"
    combined = hashlib.sha256()
    for k in ks:
        combined.update(per_k[k].encode())
    assert combined.hexdigest() == d["combined_sha256"]
    for t, pt in enumerate(pts):
        assert sums[t] == eval_host(f, pt) * eval_host(g, pt) % P
