"""CPU checks of the C ABI library: it loads, exports every symbol that
include/tlsrqi.h declares, and its host-only entry points behave (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2305_19028_b200 import build, tlsrqi
    build.build()
    return tlsrqi.lib()


def _header_symbols():
    with open(os.path.join(ROOT, "include", "tlsrqi.h")) as fh:
        txt = fh.read()
    return sorted(set(re.findall(r"TLS_API\s+[\w\s\*]*?\b(tls_\w+)\s*\(", txt)))


def test_exports_every_header_symbol(L):
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    from paper_2305_19028_b200 import tlsrqi
    assert sorted(tlsrqi.EXPORTED) == syms


def test_host_entry_points(L):
    from paper_2305_19028_b200 import tlsrqi
    assert L.tls_abi_version() == 6
    for code, name in tlsrqi.STATUS.items():
        assert tlsrqi.tls_status_string(code) == name
    o = tlsrqi.tls_rqi_opts_default()
    from oracle.rqi import RqiOptions   # defaults agree with the oracle's
    ro = RqiOptions()
    for f in ("budget_rule", "stop_rule", "max_outer", "polish", "boot", "boot_max", "op_variant",
              "breakdown_rule", "gram_chunk"):
        assert getattr(o, f) == getattr(ro, f), f
    assert o.boot_tol == ro.boot_tol and o.tol_inner == ro.tol_inner


def test_struct_layouts_match_header(L):
    from paper_2305_19028_b200 import tlsrqi
    assert C.sizeof(tlsrqi.tls_matrix_t) == 4 + 4 + 5 * 8 + 3 * 8 + 8
    assert tlsrqi.tls_info_t.sigma2.offset % 8 == 0


def test_argument_validation_without_gpu(L):
    from paper_2305_19028_b200 import tlsrqi
    M = tlsrqi.tls_matrix_t()
    M.layout, M.n, M.m_local, M.m_global, M.ld = 0, 4, 3, 3, 4   # m_global < n + 1
    assert L.tls_workspace_size(C.byref(M), 50) == 0
    M.layout = 1
    M.m_global = 10
    assert L.tls_workspace_size(C.byref(M), 50) == 0             # CSR without rowptr / colidx / vals
    M.layout, M.ld = 0, 5                                        # odd ld
    assert L.tls_workspace_size(C.byref(M), 50) == 0
    M.ld, M.vals = 4, 256
    assert L.tls_workspace_size(C.byref(M), 50) > 0


def test_ctypes_layouts_equal_the_c_compiler(L, tmp_path):
    """The binding's ctypes structures have the sizes and field offsets that gcc gives the
    header's structs (the ABI of include/tlsrqi.h, checked without a GPU)."""
    import shutil
    import subprocess
    from paper_2305_19028_b200 import tlsrqi
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {"tls_matrix_t": tlsrqi.tls_matrix_t, "tls_rqi_opts_t": tlsrqi.tls_rqi_opts_t,
               "tls_info_t": tlsrqi.tls_info_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tlsrqi.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append(f'  printf("abi %d\\n", TLSRQI_ABI_VERSION);')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        *k, v = ln.split()
        got[" ".join(k)] = int(v)
    for name, cls in structs.items():
        assert got[f"{name} size"] == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[f"{name} {f}"] == getattr(cls, f).offset, (name, f)
    assert got["abi"] == L.tls_abi_version()


def test_qr_workspace_size_without_gpu(L, monkeypatch):
    """tls_qr_workspace_size (host only): 0 for CSR, a bad u_f or nranks < 1; otherwise at
    least the fp32 (fp64 for u_f = fp64) working copy, and more with a TSQR stack (nranks or
    TLS_QR_LEAVES > 1)."""
    from paper_2305_19028_b200 import tlsrqi
    M = tlsrqi.tls_matrix_t()
    M.layout, M.n, M.m_local, M.m_global, M.ld, M.vals = 0, 64, 1000, 1000, 64, 256
    s16 = L.tls_qr_workspace_size(C.byref(M), 0, 1)
    s64 = L.tls_qr_workspace_size(C.byref(M), 3, 1)
    assert s16 >= 1000 * 64 * 4 and s64 >= 1000 * 64 * 8 and s64 > s16
    assert L.tls_qr_workspace_size(C.byref(M), 0, 4) >= s16 + 4 * 64 * 64 * 8
    assert L.tls_qr_workspace_size(C.byref(M), 7, 1) == 0
    assert L.tls_qr_workspace_size(C.byref(M), 0, 0) == 0
    monkeypatch.setenv("TLS_QR_LEAVES", "3")
    assert L.tls_qr_workspace_size(C.byref(M), 0, 1) >= s16 + 3 * 64 * 64 * 8
    M.layout = 1
    assert L.tls_qr_workspace_size(C.byref(M), 0, 1) == 0
