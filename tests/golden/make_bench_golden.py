"""Golden responses of the reference's /bench handler.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bench_golden.py

Drives the reference's own FastAPI app (service/app.py:139-167) through its
test client and records, per request, the response fields that do not depend
on timing (terms, verified) plus sha256(format_poly(product)) of the same
product built through the reference's `_resolve_pair` and `mul`.  Writes
tests/golden/bench.json.  The reference is imported only here.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

from fastapi.testclient import TestClient

from polymul.io import format_poly
from polymul.parmul import MulConfig, mul
from polymul.service import app as service
from polymul.service import models

OUT = Path(__file__).resolve().parent / "bench.json"
REQUESTS = [(1, 4, "int"), (1, 8, "int"), (1, 6, "f64"), (2, 4, "int"), (2, 5, "f64"),
            (3, 4, "int"), (3, 5, "int"), (3, 4, "f64")]


def main():
    client = TestClient(service.create_app())
    rows = []
    for example, power, coeff in REQUESTS:
        req = {"example": example, "power": power, "coeff": coeff, "threads": [1, 2],
               "mergers": ["heap", "tree"], "repetitions": 2}
        r = client.post("/bench", json=req)
        assert r.status_code == 200, r.text
        body = r.json()
        f_src, g_src = service.BENCH_EXAMPLES[example]
        f, g = service._resolve_pair(models.PolyInput(expr=f_src.format(p=power)),
                                     models.PolyInput(expr=g_src.format(p=power)), None, coeff)
        prod = mul(f, g, MulConfig())
        rows.append({"request": req, "f_terms": body["f_terms"], "g_terms": body["g_terms"],
                     "result_terms": body["result_terms"], "verified": body["verified"],
                     "n_rows": len(body["rows"]), "vars": list(f.layout.vars.names),
                     "f_sha256": hashlib.sha256(format_poly(f).encode()).hexdigest(),
                     "product_sha256": hashlib.sha256(format_poly(prod).encode()).hexdigest()})
    cap = client.post("/bench", json={"example": 1, "power": 13})
    OUT.write_text(json.dumps({"generator": "tests/golden/make_bench_golden.py",
                               "reference": "polymul 0.1.0 (/root/reference/pkg)",
                               "requests": rows,
                               "power_cap": {"status": cap.status_code, "body": cap.json()}},
                              indent=1) + "\n")
    print(f"wrote {len(rows)} bench responses to {OUT}")


if __name__ == "__main__":
    main()
