"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/nacc.h declares, and host-side validation rejects bad arguments
before any launch (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(naccx?_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2305_04966_b200 import _lib as L

    return L.lib()


def test_every_declared_symbol_is_exported(lib):
    from paper_2305_04966_b200 import _lib as L

    names = declared("nacc.h")
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
        assert n in L.SIGNATURES, f"binding lacks {n}"
    hnames = declared("nacc_harness.h")
    h = L.harness()
    for n in hnames:
        assert hasattr(h, n), n


def test_exports_are_exactly_the_abi(lib):
    """No stray C symbols: every exported nacc_* function is declared."""
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2305_04966_b200", "libnacc.so")],
                         capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r"\bT (nacc_[a-z0-9_]+)\b", out)))
    assert exported == declared("nacc.h")


def test_version_and_sizes(lib):
    from paper_2305_04966_b200 import GridSpec, MarchParams

    assert lib.nacc_abi_version() == 1
    g = GridSpec(res=128, levels=4).c()
    # fine bits + private header (occupied boxes) + macro skip mask + the fine OR / AND
    # window masks (one bit per fine cell of every level each) for window sizes 2..9 on
    # cascades, 2..5 on a single level (gridaux.cu grid_fine_win)
    assert lib.nacc_grid_bits_bytes(C.byref(g)) == (1 + 2 * 8) * (4 * 128**3 // 8) + 256 + 4 * 32**3 // 8
    g1 = GridSpec(res=128, levels=1).c()
    assert lib.nacc_grid_bits_bytes(C.byref(g1)) == (1 + 2 * 4) * (128**3 // 8) + 256 + 32**3 // 8
    g.levels = 0
    assert lib.nacc_grid_bits_bytes(C.byref(g)) == 0
    g = GridSpec(res=128).c()
    p = MarchParams(step=0.01).c()
    assert lib.nacc_sampling_occgrid_workspace_bytes(C.byref(g), C.byref(p), 1 << 18) >= (1 << 18) // 2
    assert lib.nacc_filter_workspace_bytes(1000) >= 8 + 8 * 4


def test_host_validation_rejects_before_launch(lib):
    """Invalid arguments return NACC_ERR_INVALID_ARGUMENT and set the thread-local message."""
    from paper_2305_04966_b200 import GridSpec, MarchParams

    g = GridSpec(res=16).c()
    bad_steps = [MarchParams(step=0.0), MarchParams(step=float("nan")), MarchParams(step=0.01, cone_angle=-1.0)]
    fake = C.c_void_p(4096)
    for p in bad_steps:
        pc = p.c()
        st = lib.nacc_sampling_occgrid(C.byref(g), fake, C.byref(pc), fake, fake, None, None, 10, fake, None, None,
                                       None, 0, fake, None, fake, 1 << 20, None)
        assert st == 1
        assert b"step" in lib.nacc_last_error() or b"cone" in lib.nacc_last_error()
    gl = GridSpec(res=16, levels=9).c()
    pc = MarchParams(step=0.01).c()
    st = lib.nacc_sampling_occgrid(C.byref(gl), fake, C.byref(pc), fake, fake, None, None, 10, fake, None, None, None,
                                   0, fake, None, fake, 1 << 20, None)
    assert st == 1 and b"levels" in lib.nacc_last_error()
    # workspace too small
    st = lib.nacc_sampling_occgrid(C.byref(g), fake, C.byref(pc), fake, fake, None, None, 10, fake, None, None, None,
                                   0, fake, None, fake, 8, None)
    assert st == 1 and b"workspace" in lib.nacc_last_error()
    # cone marching with per-ray anchors is unsupported
    pcone = MarchParams(step=0.01, cone_angle=0.01, max_step=1.0).c()
    st = lib.nacc_sampling_occgrid(C.byref(g), fake, C.byref(pcone), fake, fake, fake, None, 10, fake, None, None,
                                   None, 0, fake, None, fake, 1 << 24, None)
    assert st == 4
    assert lib.nacc_render_fwd(None, None, 5, None, None, None, None, 3, 1.0, None, None, None, None, None) == 1
    assert lib.nacc_render_fwd(fake, None, -1, None, None, None, None, 3, 1.0, None, None, None, None, None) == 1
    assert lib.nacc_accumulate_along_rays(fake, 3, fake, None, 3, 5, fake, None) == 1  # values NULL needs C == 1
    assert lib.nacc_importance_sample(4, 8, fake, fake, fake, 1, 0.2, 1000.0, 4, 0, 0, fake, None, None) == 1
    assert lib.nacc_importance_sample(4, 8, fake, fake, None, 0, 0.2, float("inf"), 4, 0, 0, fake, None, None) == 1
    assert lib.nacc_occgrid_update(C.byref(g), fake, fake, 0, 1.5, 0.01, 0, fake, None, fake, 1 << 20, None) == 1
    assert lib.nacc_occgrid_points(C.byref(g), 0, 0, 1, 0, 16**3 + 1, fake, None) == 1
    assert lib.nacc_filter_early_stop(fake, 4, fake, fake, fake, 10, float("nan"), fake, fake, fake, fake, 10, fake,
                                      fake, 1 << 20, None) == 1
    # rows beyond the core path (alpha compositing, combined estimator, dynamic grid, proposal loss)
    assert lib.nacc_render_weights_alpha_fwd(fake, 4, None, 10, 1.0, fake, None, None) == 1  # alphas NULL
    assert lib.nacc_render_weights_alpha_fwd(fake, 4, fake, 10, float("nan"), fake, None, None) == 1
    assert lib.nacc_render_weights_alpha_bwd(fake, 4, fake, 10, 1.0, fake, None, fake, fake, 8, None) == 1  # ws
    assert b"workspace" in lib.nacc_last_error()
    assert lib.nacc_render_weights_alpha_bwd_workspace_bytes(1000) >= 8000
    assert lib.nacc_importance_sample_ranged(4, 8, fake, fake, None, 0, None, None, 4, 0, 0, fake, None, None) == 1
    assert lib.nacc_importance_sample_ranged(4, 8, fake, fake, fake, 0, fake, fake, 4, 0, 0, fake, None, None) == 1
    assert lib.nacc_occgrid_ray_bounds(C.byref(g), fake, C.byref(pc), fake, fake, None, None, 10, None, fake, None,
                                       fake, 1 << 20, None) == 1  # t_near NULL
    assert lib.nacc_occgrid_times(C.byref(g), 0, 0, -1, 0, 10, fake, None) == 1  # negative draw
    assert lib.nacc_occgrid_times(C.byref(g), 0, 0, 0, 0, 16**3 + 1, fake, None) == 1  # range
    assert lib.nacc_max_merge(None, fake, 10, None) == 1
    assert lib.nacc_pdf_loss(4, 0, fake, fake, 8, fake, fake, 1e-7, fake, None) == 1  # nf < 1
    assert lib.nacc_pdf_loss(4, 8, fake, fake, 8, fake, fake, 0.0, fake, None) == 1  # eps <= 0
    assert lib.nacc_pdf_loss_bwd(4, 8, fake, fake, 8, fake, fake, 1e-7, None, fake, None) == 1  # g_loss NULL
    # zero-size calls succeed without launching
    assert lib.nacc_pdf_loss(0, 8, None, None, 8, None, None, 1e-7, None, None) == 0
    assert lib.nacc_max_merge(None, None, 0, None) == 0


def test_product_has_no_oracle_dependency():
    """The product package never imports, includes or links the oracle (task rule ③)."""
    pkg = os.path.join(ROOT, "paper_2305_04966_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", s, flags=re.M), f
                assert not re.search(r"#include\s+[<\"].*oracle", s), f
                assert "liboracle" not in s, f
    import subprocess

    out = subprocess.run(["ldd", os.path.join(pkg, "libnacc.so")], capture_output=True, text=True).stdout
    assert "oracle" not in out
