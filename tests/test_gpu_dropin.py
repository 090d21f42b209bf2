"""Drop-in proof against the reference's own objects and call sites.

The reference package is installed unmodified in baseline/_ref (pip install
of /root/reference; DESIGN.md records the command).  These tests:
  * pass the reference's own Polynomial objects through the GPU `mul` and
    compare with the reference's `mul` under the reference's own __eq__;
  * execute the ctypes stub of INTEGRATION.md verbatim (as polymul.gpu);
  * rewire polymul.parmul.mul and polymul.service.app.mul (app.py:30,133) and
    run the reference's acceptance criteria 3 and 8 (test_acceptance.py:129-161,
    237-256) with the reference's generators and oracle, and its FastAPI
    /multiply and /bench handlers through TestClient.
Skipped when baseline/_ref is absent (it is git-ignored; gpurun ships it)."""

from __future__ import annotations

import importlib
import json
import os
import random
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "polymul").exists(), reason="baseline/_ref not installed")]


@pytest.fixture(scope="module")
def ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    mods = {m: importlib.import_module(f"polymul.{m}") for m in ("core", "io", "parmul", "split")}
    mods["app"] = importlib.import_module("polymul.service.app")
    assert Path(mods["core"].__file__).resolve().is_relative_to(REF.resolve())
    return type("Ref", (), mods)


def _gpu():
    from paper_1303_7425_b200 import mul
    return mul


def test_reference_objects_in_and_out(ref):
    mul = _gpu()
    core, io, parmul = ref.core, ref.io, ref.parmul
    lay = core.default_layout(("x", "y", "z", "t"))
    for ctype in (int, float):
        f = io.poly_from_expr("(1+x+y+z+t)^8", lay, ctype)
        g = f + core.Polynomial.constant(lay, 1, ctype)
        p = mul(f, g)
        assert type(p) is core.Polynomial and p.layout == f.layout
        assert p == parmul.mul(f, g)  # the reference's own equality (core.py:297-300)
        p.validate()
    lay5 = core.default_layout(("x", "y", "z", "t", "u"))
    a = io.poly_from_expr("(1+x+y+2*z^2+3*t^3+5*u^5)^5", lay5)
    b = io.poly_from_expr("(1+u+t+2*z^2+3*y^3+5*x^5)^5", lay5)
    assert mul(a, b) == parmul.mul(a, b, parmul.MulConfig(l=7, c=2))
    assert mul(a, b, parmul.MulConfig(l=7, c=2, merger="tree")) == core.naive_mul(a, b)
    # split= keeps the reference semantics (products below bounds[0] not formed)
    x = core.Polynomial.variable(lay, "x")
    one_x = core.Polynomial.constant(lay, 1) + x
    sp = ref.split.SplitSet([lay.pack((1, 0, 0, 0)), core.SENTINEL])
    assert mul(one_x, one_x, split=sp) == parmul.mul(one_x, one_x, split=sp)
    # errors map onto the reference's exception types
    half = core.Polynomial(lay, [(1, (3000, 0, 0, 0))])  # x^6000 overflows the 12-bit x field
    with pytest.raises(Exception) as e1:
        parmul.mul(half, half)
    with pytest.raises(Exception) as e2:
        mul(half, half)
    assert type(e2.value).__name__ == type(e1.value).__name__ == "ExponentOverflowError"


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## The stub a maintainer adds"):]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_integration_stub_runs_verbatim(tmp_path):
    """The INTEGRATION.md stub, executed unmodified as module polymul.gpu of the
    reference package, multiplies reference objects like the reference."""
    script = tmp_path / "run_stub.py"
    script.write_text(f'''
import sys, types, json
sys.path.insert(0, {str(REF)!r})
import polymul
from polymul import core, io, parmul
mod = types.ModuleType("polymul.gpu"); mod.__package__ = "polymul"; sys.modules["polymul.gpu"] = mod
exec(compile(open({str(tmp_path / "stub.py")!r}).read(), "polymul/gpu.py", "exec"), mod.__dict__)
lay = core.default_layout(("x", "y", "z", "t"))
out = {{}}
for ctype in (int, float):
    f = io.poly_from_expr("(1+x+y+z+t)^6", lay, ctype)
    g = f + core.Polynomial.constant(lay, 1, ctype)
    out[ctype.__name__] = mod.gpu_mul(f, g) == parmul.mul(f, g)
parmul.mul = mod.gpu_mul  # the wiring INTEGRATION.md describes
h = io.eval_expr(io.parse_expr("(1+x+y)^7*(1-z+t)^3", lay.vars), lay, int, mul=mod.gpu_mul)
out["eval_expr"] = h == io.eval_expr(io.parse_expr("(1+x+y)^7*(1-z+t)^3", lay.vars), lay, int)
print(json.dumps(out))
''')
    (tmp_path / "stub.py").write_text(_stub_source())
    env = dict(os.environ, LD_LIBRARY_PATH=str(ROOT / "paper_1303_7425_b200" / "lib"))
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert json.loads(r.stdout.strip().splitlines()[-1]) == {"int": True, "float": True, "eval_expr": True}


def _safe_max_deg(m, terms, dense):
    """test_acceptance.py:48-57, restated."""
    d = 1
    while (d + 1) ** m < 2 * terms:
        d += 1
    if not dense:
        d *= 3
    cap = {1: 4000, 2: 2000, 3: 500, 4: 500, 5: 120, 6: 40, 7: 25, 8: 15}[m]
    return min(d, cap)


def test_rewired_acceptance_criterion_3(ref, monkeypatch):
    """Criterion 3 (test_acceptance.py:129-161) with polymul.parmul.mul rewired
    to the GPU: 500 random products, the reference's generator and seed, equal
    to the reference's schoolbook oracle."""
    monkeypatch.setattr(ref.parmul, "mul", _gpu())
    mul, random_sparse, naive_mul, MulConfig = ref.parmul.mul, ref.parmul.random_sparse, ref.core.naive_mul, \
        ref.parmul.MulConfig
    rng = random.Random(0xACCE97)
    l_cycle = (1, 2, 7, 64)
    merger_cycle = ("heap", "tree")
    for idx in range(500):
        m = (idx % 8) + 1
        roll = rng.random()
        if roll < 0.80:
            terms = rng.randint(1, 150)
        elif roll < 0.95:
            terms = rng.randint(150, 600)
        else:
            terms = rng.randint(600, 2000)
        terms_b = rng.randint(1, terms)
        if terms * terms_b > 400_000:
            terms_b = max(1, 400_000 // terms)
        dense = idx % 2 == 0
        a = random_sparse(rng.randrange(1 << 30), m, terms, _safe_max_deg(m, terms, dense))
        b = random_sparse(rng.randrange(1 << 30), m, terms_b, _safe_max_deg(m, terms_b, dense))
        parallel = idx % 6 == 0
        cfg = MulConfig(l=l_cycle[(idx // 6) % 4 if parallel else idx % 4], c=4 if parallel else 1,
                        merger=merger_cycle[(idx // 4) % 2])
        got = mul(a, b, cfg)
        assert type(got) is ref.core.Polynomial
        assert got == naive_mul(a, b), f"case {idx}: m={m} terms={terms}x{terms_b}"


def test_rewired_acceptance_criterion_8(ref, monkeypatch):
    """Criterion 8 (test_acceptance.py:237-256): bit-identical output for any
    worker count and merger, ints and floats; and equal to the reference's."""
    ref_mul = ref.parmul.mul
    monkeypatch.setattr(ref.parmul, "mul", _gpu())
    core, io, parmul = ref.core, ref.io, ref.parmul
    lay = core.default_layout(("x", "y", "z", "t"))
    f = io.poly_from_expr("(1+x+y+z+t)^7", lay)
    g = f + core.Polynomial.constant(lay, 1)
    fa = parmul.random_sparse(0xD0, 4, 150, 12, ctype=float)
    fb = parmul.random_sparse(0xD1, 4, 150, 12, ctype=float)
    want_int = ref_mul(f, g, parmul.MulConfig(l=16))
    want_flt = ref_mul(fa, fb, parmul.MulConfig(l=16))
    for merger in ("heap", "tree"):
        for c in (1, 2, 4, 8):
            run_int = parmul.mul(f, g, parmul.MulConfig(l=16, c=c, merger=merger))
            assert run_int.exps == want_int.exps and run_int.coeffs == want_int.coeffs
            run_flt = parmul.mul(fa, fb, parmul.MulConfig(l=16, c=c, merger=merger))
            assert run_flt.exps == want_flt.exps
            assert all(x == y for x, y in zip(run_flt.coeffs, want_flt.coeffs))


def test_rewired_service_multiply_and_bench(ref, monkeypatch):
    """The reference's FastAPI handlers with app.mul rewired (app.py:30: bound
    by name at import) give the reference's responses: /multiply result text,
    and /bench term counts with verified == True (schoolbook check, app.py:161-164)."""
    from fastapi.testclient import TestClient
    client = TestClient(ref.app.create_app())
    reqs = [{"a": {"expr": "(1+x+y+z+t)^6"}, "b": {"expr": "(1+x+y+z+t)^6+1"}},
            {"a": {"expr": "(1+x+y+2*z^2+3*t^3+5*u^5)^4"}, "b": {"expr": "(1+u+t+2*z^2+3*y^3+5*x^5)^4"},
             "options": {"coeff": "f64", "l": 7, "threads": 2}},
            {"a": {"text": "vars x y\n3 1 0\n-2 0 1\n"}, "b": {"expr": "(x-y)^5"}}]
    want = [client.post("/multiply", json=r).json() for r in reqs]
    bench_req = {"example": 2, "power": 5, "threads": [1, 2], "mergers": ["heap", "tree"], "coeff": "int"}
    want_bench = client.post("/bench", json=bench_req).json()
    monkeypatch.setattr(ref.app, "mul", _gpu())
    got = [client.post("/multiply", json=r).json() for r in reqs]
    for w, g in zip(want, got):
        assert g["result"] == w["result"] and g["result_terms"] == w["result_terms"]
    got_bench = client.post("/bench", json=bench_req).json()
    assert got_bench["result_terms"] == want_bench["result_terms"]
    assert got_bench["verified"] is True and len(got_bench["rows"]) == 4
