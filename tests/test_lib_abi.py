"""The C-ABI library loads and exports every symbol include/vf.h declares; argument validation
runs before any device work (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def vf():
    from paper_2506_00812_b200 import build as B
    B.build()
    import paper_2506_00812_b200 as vf
    vf.lib()
    return vf


def test_exports_every_declared_symbol(vf):
    hdr = open(os.path.join(ROOT, "include", "vf.h")).read()
    declared = set(re.findall(r"^\s*(?:vf_status|void|const char \*)\s*(vf_\w+)\s*\(", hdr, re.M))
    assert {"vf_build_index", "vf_search", "vf_free", "vf_last_error"} <= declared
    lib = C.CDLL(vf.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(vf.EXPORTED) == declared


def test_library_is_sm100a_native(vf):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", vf.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports / links the oracle."""
    pkg = os.path.join(ROOT, "paper_2506_00812_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower().replace("oracle/", ""), f


def _desc(vf, X, off, ids, T=2, R=2, goff=None, gids=None):
    d = vf.BuildDesc()
    d.n_points, d.dim, d.dtype = X.shape[0], X.shape[1], vf.VF_F32
    d.vectors = X.ctypes.data_as(C.c_void_p)
    d.n_labels = len(off) - 1
    d.posting_offsets = off.ctypes.data_as(C.c_void_p)
    d.posting_ids = ids.ctypes.data_as(C.c_void_p)
    d.threshold_T, d.degree_R = T, R
    if goff is not None:
        d.graph_row_offsets = goff.ctypes.data_as(C.c_void_p)
        d.graph_local_ids = gids.ctypes.data_as(C.c_void_p)
    d.world_size, d.rank, d.device = 1, 0, 0
    return d


@pytest.mark.parametrize("case", ["unsorted", "out_of_range", "hs_without_graph", "bad_graph_entry",
                                  "bad_T", "bad_dim"])
def test_build_validation_errors(vf, case):
    X = np.zeros((6, 4), np.float32)
    off = np.array([0, 3, 4], np.int64)
    ids = np.array([0, 2, 5, 1], np.int32)
    goff = np.array([0, 3, 3], np.int64)
    gids = np.array([1, 2, 0, 2, 0, 1], np.int32)
    kw = {}
    if case == "unsorted":
        ids = np.array([2, 0, 5, 1], np.int32)
    elif case == "out_of_range":
        ids = np.array([0, 2, 6, 1], np.int32)
    elif case == "hs_without_graph":
        goff, gids = None, None
    elif case == "bad_graph_entry":
        gids = np.array([1, 2, 3, 2, 0, 1], np.int32)
    elif case == "bad_T":
        kw["T"] = 0
    d = _desc(vf, X, off, ids, goff=goff, gids=gids, **kw)
    if case == "bad_dim":
        d.dim = 0
    h = C.c_void_p()
    st = vf.lib().vf_build_index(C.byref(d), C.byref(h))
    assert st == vf.VF_ERR_INVALID_ARG
    assert h.value is None
    assert len(vf.lib().vf_last_error()) > 0


def test_null_safety(vf):
    vf.lib().vf_free(None)
    st = vf.lib().vf_search(None, None, 0, None, None, None, None, None, None)
    assert st == vf.VF_ERR_INVALID_ARG


def test_serve_null_safety(vf):
    """The serving calls validate their arguments before touching a device (no GPU needed)."""
    import ctypes as C
    L = vf.lib()
    t = C.c_int64()
    assert L.vf_serve_start(None, None, 16, 0, None) == vf.VF_ERR_INVALID_ARG
    assert L.vf_serve_submit(None, None, None, 0, C.byref(t)) == vf.VF_ERR_INVALID_ARG
    assert L.vf_serve_wait(None, 0, None, None) == vf.VF_ERR_INVALID_ARG
    assert L.vf_serve_run(None, 0, None, None, None, 1, None, None) == vf.VF_ERR_INVALID_ARG
    assert L.vf_serve_info(None, None, None) == vf.VF_ERR_INVALID_ARG
    assert L.vf_serve_stop(None) == vf.VF_OK
