"""CPU-only checks of the C-ABI boundary: the library loads, exports every symbol that
include/gjinv.h declares, and its argument validation answers without touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
            names |= set(re.findall(r"\b(gj_\w+)\s*\(", txt))
    return names


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def test_library_exports_every_declared_symbol(gj):
    decl = _declared()
    assert {"gj_invert_batched", "gj_invert", "gj_det", "gj_workspace_size", "gj_status_string"} <= decl
    for name in sorted(decl):
        assert hasattr(gj.lib, name), f"{name} declared in include/ but not exported by libgjinv.so"


def test_status_strings(gj):
    for s in range(6):
        assert gj.lib.gj_status_string(s).decode().startswith("GJ_")
    assert b"sm_100a" in gj.lib.gj_version()


def test_argument_errors_need_no_gpu(gj):
    L = gj.lib
    # n < 1, negative batch, bad dtype -> GJ_ERR_ARG before any CUDA call
    assert L.gj_invert_batched(0, 0, 10, 1, 1, None, None, None, None, None, -1.0, None) == 1
    assert L.gj_invert_batched(0, 4, -1, 1, 1, None, None, None, None, None, -1.0, None) == 1
    assert L.gj_invert_batched(7, 4, 1, 1, 1, None, None, None, None, None, -1.0, None) == 1
    # batch == 0 is a no-op
    assert L.gj_invert_batched(0, 4, 0, None, None, None, None, None, None, None, -1.0, None) == 0
    # n above the batched limit -> GJ_ERR_UNSUPPORTED
    assert L.gj_invert_batched(1, 65, 1, 1, 1, None, None, None, None, None, -1.0, None) == 2
    # NULL A
    assert L.gj_invert_batched(1, 4, 3, None, None, None, None, None, None, None, -1.0, None) == 1
    assert L.gj_invert(1, 4, None, 4, None, 4, None, None, None, None, -1.0, None, 0, None) == 1


def test_workspace_size(gj):
    L = gj.lib
    assert L.gj_workspace_size(0, 32, 100, 0) == 0
    assert L.gj_workspace_size(1, 16, 1, 1) == 16 * 16 * 8


def test_no_oracle_in_product_path():
    """The product package must not import or reference oracle/."""
    pkg = os.path.join(ROOT, "paper_1401_7962_b200")
    for dp, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".h", ".cpp", ".cuh")):
                txt = open(os.path.join(dp, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "gjo_" not in txt, fn


def test_argument_errors_new_entries(gj):
    """f2-f4 entry points: the same argument contract, answered without a GPU."""
    L = gj.lib
    # full / strategy kernels: n < 1, n > 32, bad strategy, NULL A, empty batch
    assert L.gj_invert_batched_full(0, 0, 4, 1, None, None, None, None, None, None, None, -1.0, None) == 1
    assert L.gj_invert_batched_full(0, 33, 4, 1, None, None, None, None, None, None, None, -1.0, None) == 2
    assert L.gj_invert_batched_full(0, 8, 0, None, None, None, None, None, None, None, None, -1.0, None) == 0
    assert L.gj_invert_batched_pivoting(0, 8, 4, 1, None, None, None, None, None, None, None, -1.0, 3, None) == 1
    assert L.gj_invert_batched_pivoting(0, 8, 4, None, None, None, None, None, None, None, None, -1.0, 2, None) == 1
    # batched solve: nrhs < 1, NULL B / X, limits
    assert L.gj_solve_batched(0, 8, 0, 4, 1, 1, 1, None, None, None, None, -1.0, None) == 1
    assert L.gj_solve_batched(0, 8, 2, 4, 1, None, 1, None, None, None, None, -1.0, None) == 1
    assert L.gj_solve_batched(0, 8, 33, 4, 1, 1, 1, None, None, None, None, -1.0, None) == 2
    assert L.gj_solve_batched(0, 8, 2, 0, None, None, None, None, None, None, None, -1.0, None) == 0
    # single solve: bad leading dimensions, strided small system, missing workspace
    assert L.gj_solve(1, 8, 2, 1, 7, 1, 2, 1, 2, None, None, None, None, -1.0, None, 0, None) == 1
    assert L.gj_solve(1, 8, 2, 1, 9, 1, 2, 1, 2, None, None, None, None, -1.0, None, 0, None) == 2
    assert L.gj_solve(1, 100, 2, 1, 100, 1, 2, 1, 2, None, None, None, None, -1.0, None, 0, None) == 3


def test_solve_workspace_sizes(gj):
    L = gj.lib
    assert L.gj_solve_workspace_size(0, 32, 32) == 0     # the batched kernel: none
    for dt in (0, 1):
        small, big = L.gj_solve_workspace_size(dt, 100, 1), L.gj_solve_workspace_size(dt, 1000, 64)
        assert 0 < small < big


def test_large_order_limit(gj):
    """Above GJ_LARGE_MAX_N (65536) the single-matrix entries answer GJ_ERR_UNSUPPORTED."""
    L = gj.lib
    n = 65536 + 128
    assert L.gj_invert(1, n, 1, n, 1, n, None, None, None, None, -1.0, 1, 1 << 40, None) == 2
    assert L.gj_det(1, n, 1, 1, None, None, None, None, None, -1.0, 1, 1 << 40, None) == 2
    assert L.gj_solve(1, n, 1, 1, n, 1, 1, 1, 1, None, None, None, None, -1.0, 1, 1 << 40, None) == 2


def test_dist_handle_entry_points_check_arguments():
    """gj_dist_init / gj_invert_dist / gj_dist_finalize refuse bad arguments before touching
    NCCL or the GPU (include/gjinv.h)."""
    import ctypes
    import paper_1401_7962_b200 as gj
    L = gj.lib
    h = ctypes.c_void_p()
    uid = (ctypes.c_ubyte * 128)()
    assert L.gj_dist_init(0, 0, uid, 0, ctypes.byref(h)) == 1          # nranks < 1
    assert L.gj_dist_init(9, 0, uid, 0, ctypes.byref(h)) == 1          # > GJ_DIST_MAX_RANKS
    assert L.gj_dist_init(2, 2, uid, 0, ctypes.byref(h)) == 1          # rank out of range
    assert L.gj_dist_init(1, 0, None, 0, ctypes.byref(h)) == 1         # no unique id
    assert L.gj_dist_init(1, 0, uid, -1, ctypes.byref(h)) == 1         # device
    assert L.gj_dist_init(1, 0, uid, 0, None) == 1                     # no handle
    assert L.gj_invert_dist(None, 1000, None, 1, None, 1, None, None, None, None, -1.0, None) == 1
    assert L.gj_dist_finalize(None) == 0
    assert L.gj_dist_get_unique_id(None) == 1
