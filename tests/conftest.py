"""Shared fixtures.  `gpu` tests need a CUDA device and the built library;
everything else runs on the CPU (oracle vs golden vectors, host logic, ABI
symbol checks, gloo world-size-2 partition/gather)."""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import random
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"

from paper_1303_7425_b200.core import Layout, Polynomial, VarTable  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


def dec_coef(s: str, ctype):
    if ctype is int:
        return int(s)
    return float(s)


def dec_layout(d) -> Layout:
    return Layout(VarTable(tuple(d["vars"])), d["order"], tuple(d["var_bits"]),
                  d["deg_bits"] if d["order"] == "grlex" else None)


def dec_poly(d, layout, ctype) -> Polynomial:
    return Polynomial._from_sorted(layout, [int(e) for e in d["exps"]],
                                   [dec_coef(c, ctype) for c in d["coeffs"]], ctype)


def enc_coef(c) -> str:
    if isinstance(c, float):
        if math.isnan(c):
            return "nan"
        if math.isinf(c):
            return "inf" if c > 0 else "-inf"
        return repr(c)
    return str(c)


def product_digest(exps, coeffs) -> str:
    """Same format as tests/golden/make_golden.py::product_digest."""
    h = hashlib.sha256()
    for e, c in zip(exps, coeffs):
        h.update(f"{e} {enc_coef(c)}\n".encode())
    return h.hexdigest()


@lru_cache(maxsize=1)
def golden():
    return json.loads(gzip.decompress((GOLDEN / "cases.json.gz").read_bytes()))


@lru_cache(maxsize=1)
def digests():
    return json.loads((GOLDEN / "digests.json").read_text())


def golden_cases():
    out = []
    for c in golden()["cases"]:
        lay = dec_layout(c["layout"])
        ct = float if c["ctype"] == "float" else int
        a = dec_poly(c["a"], lay, ct)
        b = dec_poly(c["b"], lay, ct)
        split = None if c["split"] is None else [int(x) for x in c["split"]]
        out.append((c["name"], a, b, split, c["product"]))
    return out


def golden_case_ids():
    return [c["name"] for c in golden()["cases"]]


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return random.Random(20260811)
