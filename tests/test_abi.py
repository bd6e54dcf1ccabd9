"""C-ABI tests that need no GPU (-m "not gpu"): the library builds and loads,
exports every symbol include/occ.h declares, and rejects bad arguments on the
host before anything is enqueued (fake, never-dereferenced device pointers)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2301_09830_b200 import build as occ_build
from paper_2301_09830_b200 import occ

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "occ.h")


@pytest.fixture(scope="module")
def L():
    occ_build.build()
    return occ.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(occ_\w+)\s*\(", src, flags=re.M))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for want in ["occ_compress", "occ_decompress", "occ_allreduce_factors", "occ_send_factors",
                 "occ_recv_factors", "occ_sendrecv_factors", "occ_embed_sync", "occ_init_q", "occ_workspace_bytes",
                 "occ_comm_init", "occ_comm_split", "occ_comm_destroy", "occ_get_unique_id"]:
        assert want in names


def test_library_exports_every_declared_symbol(L):
    out = subprocess.run(["nm", "-D", "--defined-only", occ.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (occ_\w+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # the exports are plain C symbols (no C++ mangling leaks through the ABI)
    assert not re.search(r"\bT _Z\w*occ_", out)


def test_library_targets_sm100a(L):
    out = subprocess.run(["cuobjdump", "--list-elf", occ.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(L):
    assert occ.occ_status_string(0) == "OCC_OK"
    for i, name in enumerate(occ.STATUS):
        assert occ.occ_status_string(i) == name
    assert "sm_100a" in occ.occ_version()


def test_workspace_bytes(L):
    a = occ.occ_workspace_bytes(1024, 3072, 16)
    b = occ.occ_workspace_bytes(4096, 3072, 16)
    assert a > 0 and b > 0
    assert occ.occ_workspace_bytes(1024, 3072, 16, nmat=2) > a
    assert occ.occ_workspace_bytes(0, 3072, 16) == 0


FAKE = 0x7F0000000000  # 256-aligned, never dereferenced: validation fails before any launch


def fmat(off, rows, cols, ld=None, dt=occ.OCC_F32):
    return occ.occ_mat(FAKE + off, rows, cols, ld if ld is not None else cols, dt)


def compress_status(L, M, E, Q, P, R=None, r=16, flags=0, ws_bytes=None):
    R = R or occ.occ_mat(None, 0, 0, 0, 0)
    ws_bytes = occ.occ_workspace_bytes(M.rows, M.cols, r) if ws_bytes is None else ws_bytes
    return L.occ_compress(M, E, Q, P, R, r, flags, ctypes.c_void_p(FAKE + (1 << 36)), ws_bytes, None)


def good(n=256, m=512, r=16):
    MB = 1 << 30
    return fmat(0, n, m), fmat(MB, n, m), fmat(2 * MB, m, r), fmat(3 * MB, n, r)


def status_name(L, s):
    return occ.STATUS[s]


@pytest.mark.parametrize("case,expect", [
    ("rank_too_big", "OCC_ERR_RANK"),
    ("rank_unsupported", "OCC_ERR_UNSUPPORTED"),
    ("q_shape", "OCC_ERR_SHAPE"),
    ("p_shape", "OCC_ERR_SHAPE"),
    ("err_shape", "OCC_ERR_SHAPE"),
    ("cols_not_mult8", "OCC_ERR_SHAPE"),
    ("misaligned", "OCC_ERR_ALIGN"),
    ("bad_ld", "OCC_ERR_ALIGN"),
    ("q_bf16", "OCC_ERR_DTYPE"),
    ("alias", "OCC_ERR_ALIAS"),
    ("workspace", "OCC_ERR_WORKSPACE"),
    ("null_err", "OCC_ERR_INVALID_ARG"),
    ("empty", "OCC_ERR_SHAPE"),
])
def test_compress_argument_errors(L, case, expect):
    M, E, Q, P = good()
    kw = {}
    if case == "rank_too_big":
        M, E, Q, P = good(n=8, m=64, r=16)
    elif case == "rank_unsupported":
        Q, P = fmat(2 << 30, 512, 12), fmat(3 << 30, 256, 12)
        kw["r"] = 12
    elif case == "q_shape":
        Q = fmat(2 << 30, 511, 16)
    elif case == "p_shape":
        P = fmat(3 << 30, 256, 8)
    elif case == "err_shape":
        E = fmat(1 << 30, 256, 520)
    elif case == "cols_not_mult8":
        M, E, Q, P = fmat(0, 256, 500, ld=504), fmat(1 << 30, 256, 500, ld=504), fmat(2 << 30, 500, 16), fmat(3 << 30, 256, 16)
    elif case == "misaligned":
        M = occ.occ_mat(FAKE + 4, 256, 512, 512, occ.OCC_F32)
    elif case == "bad_ld":
        M = fmat(0, 256, 512, ld=514)
    elif case == "q_bf16":
        Q = fmat(2 << 30, 512, 16, dt=occ.OCC_BF16)
    elif case == "alias":
        E = fmat(4096, 256, 512)
    elif case == "workspace":
        kw["ws_bytes"] = 1024
    elif case == "null_err":
        E = occ.occ_mat(None, 0, 0, 0, 0)
    elif case == "empty":
        M = fmat(0, 0, 512)
    s = compress_status(L, M, E, Q, P, **kw)
    assert status_name(L, s) == expect, L.occ_last_error().decode()
    assert L.occ_last_error().decode()


def test_no_ef_allows_null_err(L):
    M, _, Q, P = good()
    E = occ.occ_mat(None, 0, 0, 0, 0)
    s = compress_status(L, M, E, Q, P, flags=occ.OCC_NO_EF, ws_bytes=16)
    assert status_name(L, s) == "OCC_ERR_WORKSPACE"   # got past the err check


def test_decompress_argument_errors(L):
    P, Q, out = fmat(0, 256, 16), fmat(1 << 30, 512, 16), fmat(2 << 30, 256, 512)
    assert status_name(L, L.occ_decompress(P, fmat(1 << 30, 512, 8), out, None)) == "OCC_ERR_SHAPE"
    assert status_name(L, L.occ_decompress(P, Q, fmat(4096, 256, 512), None)) == "OCC_ERR_ALIAS"


def test_allreduce_factors_rank_mismatch(L):
    M1, E1, Q1, P1 = good()
    arr = occ.occ_mat * 2
    rs = (ctypes.c_int * 2)(16, 8)
    s = L.occ_allreduce_factors(2, arr(M1, M1), arr(E1, E1), arr(Q1, Q1), arr(P1, P1), rs, 0.5, 0, None,
                                ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_RANK"


def test_allreduce_factors_rejects_wire_bf16(L):
    """OCC_WIRE_BF16 (reading C7) is defined for the PP send / recv calls only:
    the DP exchange sums factors, so occ_allreduce_factors refuses it."""
    M1, E1, Q1, P1 = good()
    arr = occ.occ_mat * 1
    rs = (ctypes.c_int * 1)(16)
    s = L.occ_allreduce_factors(1, arr(M1), arr(E1), arr(Q1), arr(P1), rs, 1.0, occ.OCC_WIRE_BF16, None,
                                ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_UNSUPPORTED"


def test_comm_null_handles(L):
    M, E, Q, P = good()
    s = L.occ_send_factors(M, E, Q, P, 16, 1, 0, None, ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_INVALID_ARG"
    s = L.occ_sendrecv_factors(M, E, Q, P, 16, 1, M, P, Q, 1, 0, None, ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_INVALID_ARG"
    assert L.occ_comm_destroy(None) == 0
    h = ctypes.c_void_p()
    assert status_name(L, L.occ_comm_wrap(ctypes.byref(h), None)) == "OCC_ERR_INVALID_ARG"


def test_python_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(occ, "_lib", None)
    monkeypatch.setattr(occ, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError):
        occ.lib()


def test_link_argument_errors(L):
    """occ_link (f1): null handles and bad peers are rejected on the host."""
    h = ctypes.c_void_p()
    assert status_name(L, L.occ_link_open(None, 0, 0, 16, 16, 4, ctypes.byref(h))) == "OCC_ERR_INVALID_ARG"
    assert L.occ_link_close(None) == 0
    M, E, Q, P = good()
    s = L.occ_sendrecv_factors_link(M, E, Q, P, 16, M, P, Q, 0, None, ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_INVALID_ARG"
    assert {"occ_link_open", "occ_link_close", "occ_sendrecv_factors_link"} <= set(declared_functions())


def test_dplink_argument_errors(L):
    """occ_dplink (f1, DP): null handles are rejected on the host."""
    h = ctypes.c_void_p()
    assert status_name(L, L.occ_dplink_open(None, 1024, ctypes.byref(h))) == "OCC_ERR_INVALID_ARG"
    assert L.occ_dplink_close(None) == 0
    M, E, Q, P = good()
    arr = occ.occ_mat * 1
    rs = (ctypes.c_int * 1)(16)
    s = L.occ_allreduce_factors_link(1, arr(M), arr(E), arr(Q), arr(P), rs, ctypes.c_float(1.0), 0, None,
                                     ctypes.c_void_p(FAKE), 1 << 30, None)
    assert status_name(L, s) == "OCC_ERR_INVALID_ARG"
    assert status_name(L, L.occ_dplink_allreduce(None, ctypes.c_void_p(FAKE), ctypes.c_void_p(FAKE), 16, None)) == \
        "OCC_ERR_INVALID_ARG"
    assert {"occ_dplink_open", "occ_dplink_close", "occ_dplink_allreduce",
            "occ_allreduce_factors_link"} <= set(declared_functions())
