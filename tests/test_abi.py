"""CPU-only checks of the C-ABI boundary: libgsicp.so builds, loads, exports every function
include/gsicp.h declares, sizes workspaces, and rejects bad arguments before launching anything."""
import ctypes as C
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_2403_12550_b200 import _build

    _build.build()
    import paper_2403_12550_b200 as g

    return g


def header_functions():
    src = open(os.path.join(ROOT, "include", "gsicp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsicp_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(g):
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(g.lib(), n), n
    assert set(names) == set(g.EXPORTED)
    assert g.lib().gsicp_abi_version() == 1


def test_workspace_sizes(g):
    L = g.lib()
    assert L.gsicp_backproject_workspace_size(680, 1200, 4) >= 256
    assert L.gsicp_backproject_workspace_size(0, 1200, 4) == 0
    a = L.gsicp_covariances_workspace_size(51000, 1)
    b = L.gsicp_covariances_workspace_size(51000, 5)
    assert 0 < a < b
    assert L.gsicp_covariances_workspace_size(51000, 9) == 0
    assert L.gsicp_build_target_workspace_size(10 ** 6) > 10 ** 6 * 48
    assert L.gsicp_align_workspace_size(51000) > 51000 * 4
    for s in range(8):
        assert L.gsicp_status_string(s)


def test_invalid_arguments_rejected_without_gpu(g):
    L = g.lib()
    K = g.Intrinsics(600.0, 600.0, 599.5, 339.5)
    st = L.gsicp_backproject_downsample(None, 680, 1200, 1200, K, 4, 0.1, 10.0, None, 0, None, None, 0, None)
    assert st == g.ERR_INVALID_ARGUMENT and b"null" in L.gsicp_last_error()
    fake = C.c_void_p(0x100000)
    st = L.gsicp_backproject_downsample(fake, 680, 1200, 1000, K, 4, 0.1, 10.0, fake, 51000, fake, fake, 1 << 20,
                                        None)
    assert st == g.ERR_INVALID_ARGUMENT  # pitch < W
    st = L.gsicp_backproject_downsample(fake, 680, 1200, 1200, K, 4, 0.1, 10.0, fake, 100, fake, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT  # cap too small
    st = L.gsicp_covariances(fake, fake, 100, 33, 2, 1e-3, 0.01, 1, fake, fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT  # k > 32
    st = L.gsicp_covariances(fake, fake, 100, 20, 7, 1e-3, 0.01, 1, fake, fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT  # bad mode
    st = L.gsicp_covariances(fake, fake, 100, 20, 2, 1e-3, 0.01, 1, fake, fake, None, fake, 16, None)
    assert st == g.ERR_WORKSPACE_TOO_SMALL
    src = g._Cloud(fake, fake, fake, fake, 100)
    tgt = g._Target()
    p = g.align_params()
    T = (C.c_double * 16)()
    S = g.AlignStats()
    st = L.gsicp_align(C.byref(src), C.byref(tgt), T, C.byref(p), T, C.byref(S), fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT  # target not built
    p.max_iters = 0
    st = L.gsicp_align_async(C.byref(src), C.byref(tgt), fake, C.byref(p), fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT


def test_product_has_no_oracle_or_cpu_fallback():
    """The product package must not import the oracle or carry a CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2403_12550_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_new_entry_points_reject_bad_arguments(g):
    """Argument validation of the image-window / sampled-row / sequence / graph entry points."""
    L = g.lib()
    K = g.Intrinsics(600.0, 600.0, 599.5, 339.5)
    fake = C.c_void_p(0x100000)
    assert L.gsicp_covariances_image_workspace_size(51000, 4, 680, 1200, 4) > L.gsicp_covariances_workspace_size(51000, 4)
    assert L.gsicp_covariances_image_workspace_size(51000, 4, 0, 1200, 4) == 0
    st = L.gsicp_covariances_image(None, fake, 100, 680, 1200, 4, K, 20, g.REG_ELLIPSE, 1e-3, 0.02, 4, fake, fake,
                                   None, None, fake, 1 << 30, None, None)
    assert st == g.ERR_INVALID_ARGUMENT
    st = L.gsicp_covariances_image(fake, fake, 100, 680, 1200, 4, K, 33, g.REG_ELLIPSE, 1e-3, 0.02, 4, fake, fake,
                                   None, None, fake, 1 << 30, None, None)
    assert st == g.ERR_INVALID_ARGUMENT and b"k must be" in L.gsicp_last_error()
    st = L.gsicp_backproject_lattice(fake, 2, 680, 1200, 1200, K, 4, 0.1, 10.0, fake, 51000, fake, fake, fake, 1 << 20,
                                     None)
    assert st == g.ERR_INVALID_ARGUMENT  # rows_sampled must be 0 or 1
    st = L.gsicp_upload_sampled_rows(None, fake, 680, 1200, 1200, 4, None)
    assert st == g.ERR_INVALID_ARGUMENT
    st = L.gsicp_pose_push(fake, fake, fake, None, 4, None)
    assert st == g.ERR_INVALID_ARGUMENT  # trajectory without a counter
    assert L.gsicp_pose_predict(None, fake, None) == g.ERR_INVALID_ARGUMENT
    assert L.gsicp_graph_launch(None, None) == g.ERR_INVALID_ARGUMENT
    assert L.gsicp_graph_destroy(None) == g.OK
    E = L.gsicp_export_gaussians
    assert E(fake, fake, fake, fake, 100, None, 1.5, 1.0, None, fake, None, fake, None, None, 0, None) \
        == g.ERR_INVALID_ARGUMENT  # null quats_out
    st = E(fake, fake, fake, fake, 100, None, 1.5, 0.0, None, fake, fake, fake, None, None, 0, None)
    assert st == g.ERR_INVALID_ARGUMENT and b"c > 0" in L.gsicp_last_error()
    assert E(fake, fake, fake, fake, 0, None, 1.5, 1.0, None, fake, fake, fake, None, None, 0, None) \
        == g.ERR_INVALID_ARGUMENT
    st = E(fake, fake, fake, fake, 100, None, 1.5, 1.0, fake, fake, fake, fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT and b"d_m_out" in L.gsicp_last_error()
    st = E(fake, fake, fake, fake, 100000, None, 1.5, 1.0, fake, fake, fake, fake, fake, C.c_void_p(0x100000), 16, None)
    assert st == g.ERR_WORKSPACE_TOO_SMALL
    assert L.gsicp_export_workspace_size(100000) >= 4 * (100000 // 256)
    Bmax = L.gsicp_align_batch_max()
    assert Bmax >= 8
    st = L.gsicp_align_batch_async(fake, 0, fake, fake, fake, fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT and b"B must be" in L.gsicp_last_error()
    st = L.gsicp_align_batch_async(fake, Bmax + 1, fake, fake, fake, fake, None, fake, 1 << 20, None)
    assert st == g.ERR_INVALID_ARGUMENT
    assert L.gsicp_align_batch_async(None, 2, fake, fake, fake, fake, None, fake, 1 << 20, None) \
        == g.ERR_INVALID_ARGUMENT
