"""The C-ABI library loads and exports exactly what include/kairos_b200.h declares
(CPU: no compute calls), and the ctypes mirrors match the C structs."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "kairos_b200.h"


def declared():
    return sorted(set(re.findall(r"KR_API\s+[\w\s\*]+?\b(kr_\w+)\s*\(", HEADER.read_text())))


def test_library_built_and_exports_header_symbols():
    from paper_2605_11381_b200 import _lib
    lib = _lib.load()
    names = declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.EXPORTED) == names
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(set(re.findall(r" T (kr_\w+)", out)))
    assert exported == names


def test_library_is_sm100a():
    from paper_2605_11381_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points():
    from paper_2605_11381_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.kr_version()
    assert lib.kr_status_string(0) == b"ok"
    assert lib.kr_workspace_bytes(1 << 20) > 64 * (1 << 20)
    # argument validation happens before any device work
    assert lib.kr_horizon_confidence(None, 0, 4, 1, 8, 1.4, 1, None, None, 0, None) == _lib.KR_EINVAL
    assert lib.kr_horizon_divergence(None, None, 0, 4, 1, 8, 8, 7, None, None, None, 0.0, None,
                                     None, 0, None) == _lib.KR_EINVAL
    assert lib.kr_horizon_static(0, 8, 3, None, None) == _lib.KR_OK
    prev = lib.kr_get_dot_order()
    assert lib.kr_set_dot_order(7) == _lib.KR_EINVAL and lib.kr_get_dot_order() == prev
    assert lib.kr_set_dot_order(1) == _lib.KR_OK and lib.kr_get_dot_order() == 1
    assert lib.kr_set_dot_order(prev) == _lib.KR_OK


@pytest.mark.parametrize("env,expect", [({"OPENBLAS_CORETYPE": "Haswell"}, "haswell"),
                                        ({"OPENBLAS_CORETYPE": "Zen"}, "haswell"),
                                        ({"OPENBLAS_CORETYPE": "SkylakeX"}, "skylakex"),
                                        ({"KR_DOT_ORDER": "haswell"}, "haswell")])
def test_dot_order_follows_numpy_blas_core(env, expect):
    """The exact cosines take the ddot order of the OpenBLAS core numpy runs
    in the process (threadpoolctl), unless KR_DOT_ORDER overrides it."""
    import os
    import sys
    code = ("from paper_2605_11381_b200 import _lib\n"
            "lib = _lib.load()\n"
            "print(_lib._dot_order_choice()[0], lib.kr_get_dot_order())")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         env={**os.environ, **env}, check=True).stdout.split()
    assert out == [expect, str(_order_code(expect))]


def _order_code(name):
    return {"skylakex": 0, "haswell": 1}[name]


def test_struct_layouts_match_header():
    from paper_2605_11381_b200 import _lib
    assert ctypes.sizeof(_lib.KrFleet) == 8 * 12
    assert ctypes.sizeof(_lib.KrSched) == 4 * 4 + 8 * 6
    src = ROOT / "tests" / "_layout.c"
    src.write_text('#include "kairos_b200.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   'int main(){printf("%zu %zu %zu %zu\\n", sizeof(kr_fleet), sizeof(kr_sched),'
                   ' offsetof(kr_sched, issued_base), sizeof(kr_key));return 0;}\n')
    exe = ROOT / "tests" / "_layout"
    try:
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    finally:
        src.unlink(missing_ok=True)
        exe.unlink(missing_ok=True)
    assert [int(x) for x in out] == [ctypes.sizeof(_lib.KrFleet), ctypes.sizeof(_lib.KrSched),
                                     _lib.KrSched.issued_base.offset, 16]


def test_no_oracle_on_product_path():
    pkg = ROOT / "paper_2605_11381_b200"
    for p in pkg.rglob("*.py"):
        txt = p.read_text()
        assert "oracle" not in txt.replace("oracle/", ""), p
