"""The /bench harness mirror (reference service/app.py:139-167)
against golden responses recorded from the reference's own handler
(tests/golden/make_bench_golden.py).  Request validation and the schoolbook
`naive_mul` run on the CPU; the products themselves need the GPU."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from conftest import golden_cases, product_digest
from paper_1303_7425_b200 import io
from paper_1303_7425_b200.benchharness import BenchInputError, run_bench
from paper_1303_7425_b200.core import naive_mul

BENCH = json.loads((Path(__file__).resolve().parent / "golden" / "bench.json").read_text())


def test_power_cap_matches_reference_message():
    want = BENCH["power_cap"]
    assert want["status"] == 400 and want["body"]["error"] == "parse"
    with pytest.raises(BenchInputError) as exc:
        run_bench(1, 13)
    assert str(exc.value) == want["body"]["message"]


@pytest.mark.parametrize("bad", [dict(example=4), dict(example=1, coeff="f32"),
                                 dict(example=1, mergers=["quick"]), dict(example=1, power=0)])
def test_rejected_requests(bad):
    with pytest.raises(BenchInputError):
        run_bench(**bad)


@pytest.mark.parametrize("case", [c for c in golden_cases() if c[1].n * c[2].n <= 20000][:25],
                         ids=lambda c: c[0])
def test_naive_mul_matches_reference_products(case):
    _, a, b, split, want = case
    if split is not None:
        pytest.skip("naive_mul has no split argument")
    p = naive_mul(a, b)
    assert p.n == want["n"]
    if a.ctype is int:
        assert product_digest(p.exps, p.coeffs) == want["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("entry", BENCH["requests"],
                         ids=lambda e: "ex{example}-p{power}-{coeff}".format(**e["request"]))
def test_bench_responses_match_reference(entry):
    r = entry["request"]
    body = run_bench(r["example"], r["power"], threads=r["threads"], mergers=r["mergers"],
                     repetitions=r["repetitions"], coeff=r["coeff"])
    for k in ("f_terms", "g_terms", "result_terms", "verified"):
        assert body[k] == entry[k], k
    assert len(body["rows"]) == entry["n_rows"]
    assert [(x["merger"], x["threads"], x["repetition"]) for x in body["rows"]] == [
        (m, t, k) for m in r["mergers"] for t in r["threads"] for k in range(r["repetitions"])]
    assert all(x["time_ms"] > 0 for x in body["rows"])


@pytest.mark.gpu
@pytest.mark.parametrize("entry", BENCH["requests"],
                         ids=lambda e: "ex{example}-p{power}-{coeff}".format(**e["request"]))
def test_bench_products_match_reference_digests(entry):
    from paper_1303_7425_b200 import MulConfig, mul
    from paper_1303_7425_b200.expr import bench_pair
    r = entry["request"]
    ctype = float if r["coeff"] == "f64" else int
    exact = MulConfig(float_ordered=True)
    f, g = bench_pair(r["example"], r["power"], ctype, mul=lambda a, b: mul(a, b, exact))
    assert list(f.layout.vars.names) == entry["vars"]
    assert io.poly_digest(f) == entry["f_sha256"]
    p = mul(f, g, exact)
    assert io.poly_digest(p) == entry["product_sha256"]
    assert io.text_digest(p) == entry["product_sha256"]
