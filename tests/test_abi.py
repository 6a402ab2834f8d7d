"""The C-ABI library loads and exports every symbol include/aqr.h declares; host-side argument
validation works without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import pytest

import paper_2602_21600_b200 as aqr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "aqr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aqr_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for f in ["aqr_encode", "aqr_upload_index", "aqr_search", "aqr_rerank", "aqr_merge_topk"]:
        assert f in names


def test_library_exports_every_declared_symbol():
    lib = aqr.lib()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(aqr.EXPORTS) <= set(_declared())


def test_version_and_sm100a_build():
    assert b"sm_100a" in aqr.lib().aqr_version()
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {aqr.lib_path()} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_host_validation_without_gpu():
    lib = aqr.lib()
    p = aqr.make_params(10, 64, 21, 21)
    st = lib.aqr_search(None, None, C.c_int64(1), C.c_int64(1), C.byref(p), None, None, None, None,
                        C.c_size_t(0), None)
    assert st == 1 and b"index null" in lib.aqr_last_error()
    bad = aqr.make_params(10, 16, 21, 21)  # ef < n_coarse
    st = lib.aqr_search(C.c_void_p(1), None, C.c_int64(1), C.c_int64(1), C.byref(bad), None, None, None, None,
                        C.c_size_t(0), None)
    assert st == 1 and b"ef >= n_coarse" in lib.aqr_last_error()
    st = lib.aqr_merge_topk(None, None, C.c_int32(0), C.c_int64(1), C.c_int32(5), None, None, None)
    assert st == 1 and b"n_lists" in lib.aqr_last_error()
    st = lib.aqr_encode(None, C.c_int64(1), C.c_int32(1), C.c_int64(1), None, None, None, None)
    assert st == 1
    st = lib.aqr_upload_index(None, None, None)
    assert st == 1


def test_upload_validation_rejects_bad_graph():
    lib = aqr.lib()
    import numpy as np
    n, M = 4, 2
    adj0 = np.full((n, 2 * M), -1, np.int32)
    adj0[0, 0] = 7  # out of range
    uo = np.full(n, -1, np.int64)
    D = aqr.IndexDesc()
    D.n, D.d, D.metric, D.codes, D.d_pad, D.base, D.ld_base = n, 3, 0, 1, 16, 1, 3
    D.min_j, D.scale_j, D.M, D.max_level, D.entry_point = 1, 1, M, 0, 0
    D.adj0, D.upper_off, D.adj_upper, D.upper_rows, D.layout = adj0.ctypes.data, uo.ctypes.data, None, 0, 0
    h = C.c_void_p()
    assert lib.aqr_upload_index(C.byref(D), C.byref(h), None) == 1
    assert b"adj0 id out of range" in lib.aqr_last_error()


def test_product_fails_loudly_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(aqr.AqrError):
        aqr.encode(torch.zeros(4, 3), sample_idx=torch.zeros(2, dtype=torch.int32))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_21600_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "aqr_oracle" not in s, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            s = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2602_21600_b200", s, re.M), f
            assert not re.search(r'^\s*#\s*include\s*"[^"]*(csrc|aqr\.h|aqr_internal)', s, re.M), f


def test_version_carries_the_source_hash():
    """build.py stamps the sources' hash into the library; build() rebuilds when it differs."""
    from paper_2602_21600_b200 import build as B
    _, deps = B._aqr_deps()
    digest = B.src_hash(deps, B.NVCC_FLAGS)
    assert aqr.lib().aqr_version().decode().endswith(f"src:{digest}")
    assert B._stamped(B.LIB_AQR, digest)


def _desc(adj0, upper_off, adj_upper, M, max_level=0, entry=0):
    import numpy as np
    D = aqr.IndexDesc()
    n = adj0.shape[0]
    D.n, D.d, D.metric, D.id_base = n, 4, 0, 0
    D.codes, D.d_pad, D.base, D.ld_base = 16, 16, 16, 4  # never dereferenced: validation comes first
    D.min_j, D.scale_j = 16, 16
    D.M, D.max_level, D.entry_point = M, max_level, entry
    D._keep = (np.ascontiguousarray(adj0, np.int32), np.ascontiguousarray(upper_off, np.int64),
               np.ascontiguousarray(adj_upper, np.int32))
    D.adj0 = D._keep[0].ctypes.data
    D.upper_off = D._keep[1].ctypes.data
    D.adj_upper = D._keep[2].ctypes.data if adj_upper.size else None
    D.upper_rows = adj_upper.shape[0] if adj_upper.size else 0
    D.layout = 0
    return D


@pytest.mark.parametrize("case", ["dup0", "self0", "dup_up", "self_up"])
def test_upload_rejects_repeated_and_self_neighbours(case):
    """aqr_upload_index (include/aqr.h): a row listing a neighbour twice or its own node is an
    argument error (AQR_E_INVALID), found on the host before any device work."""
    import numpy as np
    lib = aqr.lib()
    adj0 = np.array([[1, 2, -1, -1], [0, 2, -1, -1], [0, 1, 3, -1], [2, -1, -1, -1]], np.int32)
    upper_off = np.array([0, -1, 2, -1], np.int64)   # node 0: layers 1-2 (rows 0, 1); node 2: layer 1 (row 2)
    adj_upper = np.array([[2, -1], [-1, -1], [0, -1]], np.int32)
    if case == "dup0":
        adj0[2, 3] = 1
    elif case == "self0":
        adj0[3, 1] = 3
    elif case == "dup_up":
        adj_upper[0, 1] = 2
    elif case == "self_up":
        adj_upper[1, 0] = 0  # row 1 is node 0's layer-2 row
    D = _desc(adj0, upper_off, adj_upper, M=2, max_level=2, entry=0)
    h = C.c_void_p()
    st = lib.aqr_upload_index(C.byref(D), C.byref(h), None)
    msg = lib.aqr_last_error().decode()
    assert st == 1, msg
    assert ("twice" in msg) if case.startswith("dup") else ("own node" in msg), msg
