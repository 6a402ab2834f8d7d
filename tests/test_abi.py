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
