"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
entry point include/qcb200.h declares; ctypes struct sizes match the C header."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2503_06545_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qcb200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qcb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2503_06545_b200 import build_native
        build_native.build()
    return N.lib()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(N.EXPORTED) == set(names)


def test_struct_layouts_match_header(tmp_path):
    """Compile a tiny C program printing sizeof/offsetof of the ABI structs."""
    structs = ["QcbGemm", "QcbGemmF64", "QcbHeadGemm", "QcbActQuant", "QcbWeightPrep", "QcbLnMod",
               "QcbAttention", "QcbAttentionBf16", "QcbDdpm", "QcbFeat", "QcbThresholds", "QcbPolicyVideo"]
    prog = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
            "int main(void){"]
    for s in structs:
        prog.append(f'printf("{s} %zu\\n", sizeof({s}));')
    prog.append('printf("last %zu\\n", offsetof(QcbPolicyVideo, v));')
    prog.append("return 0;}")
    c = tmp_path / "sz.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-o", str(exe), str(c)], check=True)
    out = dict(line.split() for line in subprocess.check_output([str(exe)]).decode().splitlines())
    for s in structs:
        assert int(out[s]) == ctypes.sizeof(getattr(N, s)), s
    assert int(out["last"]) == N.QcbPolicyVideo.v.offset


def test_version_string(lib):
    assert b"sm_100a" in lib.qcb_version()


def test_status_mapping():
    from paper_2503_06545_b200.errors import ConfigurationError, DimensionError
    with pytest.raises(DimensionError):
        N.check(N.QCB_ERR_DIM, "x")
    with pytest.raises(ConfigurationError):
        N.check(N.QCB_ERR_OVERFLOW, "x")
    with pytest.raises(ValueError):
        N.check(N.QCB_ERR_VALUE, "x")
    with pytest.raises(TypeError):
        N.check(N.QCB_ERR_TYPE, "x")
    N.check(N.QCB_OK, "x")
