"""The C ABI library loads and exports every symbol include/polymul_b200.h
declares; the ctypes mirrors match the C struct layouts (no GPU needed, no
compute calls)."""

from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1303_7425_b200 import _native as N
from paper_1303_7425_b200.build import LIB, build

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "polymul_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(pgpu_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_exports():
    assert declared_functions() == sorted(N.EXPORTS)


def test_library_builds_and_exports_every_symbol():
    lib_path = build()
    assert lib_path == LIB and LIB.exists()
    lib = C.CDLL(str(LIB))
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_ctypes_struct_layouts_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu\\n", sizeof(pgpu_layout), sizeof(pgpu_poly), sizeof(pgpu_options), sizeof(pgpu_result), sizeof(pgpu_text));
  printf("%zu %zu %zu %zu\\n", offsetof(pgpu_options, lo), offsetof(pgpu_options, stream), offsetof(pgpu_result, phase_ms), offsetof(pgpu_options, range_pairs));
  return 0;
}}''')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(x) for x in lines[0].split()]
    assert sizes == [C.sizeof(N.Layout), C.sizeof(N.Poly), C.sizeof(N.Options), C.sizeof(N.Result),
                     C.sizeof(N.Text)]
    offs = [int(x) for x in lines[1].split()]
    assert offs == [N.Options.lo.offset, N.Options.stream.offset, N.Result.phase_ms.offset,
                    N.Options.range_pairs.offset]


def test_library_answers_without_a_gpu():
    lib = N.load()
    assert lib.pgpu_abi_version() == 3
    assert lib.pgpu_device_count() >= 0
    o = N.default_options()
    assert o.hi == (1 << 64) - 1 and o.lo == 0 and o.coef_kind == N.F64
