"""GPU parity: the CUDA path (through the C ABI via the thin binding) against
the fp64 oracle on identical seeded inputs.

Bars (BASELINE.json north_star):
  counts, packed_info, ray_id: bit-exact;  t0/t1: bit-exact (<= 1 ulp allowed);
  early-stop cut: bit-exact outside the tie band |S - L| < 1e-9 L;
  T, α, w: abs 1e-5;  color/opacity/depth: |Δ| <= 1e-4 |ref| + 1e-6;
  g_σ, g_rgb: |Δ| <= 1e-3 (|ref| + 1e-3 max_ray |ref|);
  resampled edges: backward error <= 1e-6, monotone, |Δs| <= 1e-5 where the
  CDF slope >= 1e-2;  grid density and bits: bit-exact.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

L_EPS = -math.log(float(np.float32(1e-4)))


@pytest.fixture(scope="module")
def N():
    import torch

    import __graft_entry__

    __graft_entry__.build()
    import paper_2305_04966_b200 as N

    torch.cuda.init()
    return N


def cuda(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def gpu_march(N, occ, levels, res, roi, o, d, **kw):
    t_min = kw.pop("t_min", None)
    t_max = kw.pop("t_max", None)
    capacity = kw.pop("capacity", None)
    grid = N.GridSpec(roi=tuple(roi), res=res, levels=levels)
    bits = N.prepare_bits(grid, cuda(W.pack_bits(occ).view(np.int32)))
    p = N.MarchParams(**kw)
    s = N.sampling_occgrid(cuda(o), cuda(d), grid, bits, p, None if t_min is None else cuda(t_min),
                           None if t_max is None else cuda(t_max), capacity=capacity)
    return (s.packed_info.cpu().numpy(), s.t0.cpu().numpy(), s.t1.cpu().numpy(), s.ray_id.cpu().numpy())


def assert_march_equal(gpu, ref):
    pg, g0, g1, gr = gpu
    pr, r0, r1, rr = ref
    assert np.array_equal(pg, pr), f"packed_info differs in {np.sum(np.any(pg != pr, axis=1))} rays"
    assert np.array_equal(gr, rr)
    assert np.array_equal(g0, r0) and np.array_equal(g1, r1)


def random_rays(n, rng, lo=-0.5, hi=0.5):
    c, w = (lo + hi) / 2, hi - lo
    o = c + rng.normal(size=(n, 3)) * w * 1.5
    d = c + rng.uniform(-0.6, 0.6, (n, 3)) * w - o
    o[0], d[0] = [lo - 0.5 * w, c + 0.1 * w, c], [1, 0, 0]
    o[1], d[1] = [c, c, c], [0.3, -0.5, 0.8]
    o[2], d[2] = [lo - 0.5 * w, lo, c], [1, 0, 0]
    o[3], d[3] = [lo - 0.5 * w, hi, c], [1, 0, 0]
    o[4], d[4] = [c, c, hi + w], [0, 0, -1]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o.astype(np.float32), d.astype(np.float32)


# ============================================================================ march
def test_march_cfg1(N):
    c = W.cfg1()
    ref = O.march(c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step)
    assert_march_equal(gpu_march(N, c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step), ref)


@pytest.mark.parametrize("levels,res,cone,strat,tminmax", [
    (1, 4, 0, 0, 0), (1, 16, 0, 1, 0), (2, 8, 0, 0, 1), (3, 13, 0, 1, 1), (1, 8, 1, 0, 0), (3, 8, 1, 0, 0),
    (4, 16, 1, 0, 1)])
def test_march_random_grids(N, levels, res, cone, strat, tminmax):
    rng = np.random.default_rng(10 * levels + res + cone + 100 * strat)
    o, d = random_rays(3000, rng)
    occ = (rng.random(levels * res**3) < 0.3).astype(np.uint8)
    kw = dict(step=float(np.float32(0.0071)), stratified=strat, seed=1234)
    if cone:
        kw.update(cone_angle=float(np.float32(1 / 128)), max_step=float(np.float32(0.05)), near=0.02)
    t_min = t_max = None
    if tminmax:
        t_max = rng.uniform(0.5, 3.0, len(o)).astype(np.float32)
        if not cone:
            t_min = rng.uniform(0.0, 0.5, len(o)).astype(np.float32)
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    ref = O.march(occ, levels, res, roi, o, d, t_min=t_min, t_max=t_max, **kw)
    kw_g = dict(kw)
    if "near" in kw_g:
        kw_g["near_plane"] = kw_g.pop("near")
    got = gpu_march(N, occ, levels, res, roi, o, d, t_min=t_min, t_max=t_max, **kw_g)
    assert_march_equal(got, ref)
    got = gpu_march(N, occ, levels, res, roi, o, d, t_min=t_min, t_max=t_max, capacity=len(ref[1]) + 1, **kw_g)
    assert_march_equal(got, ref)
    assert ref[0][:, 1].sum() > 1000


@pytest.mark.parametrize("res,near,strat", [(16, 0.0, 0), (16, 2.0**-60, 0), (13, 2.0**-60, 0), (16, 0.0, 1)])
def test_march_far_origin_wide_indices(N, res, near, strat):
    """Lattice indices in [2^22, 2^24): origins 4e3-1.6e4 away at Δt = 2^-10, where
    k + 1/2 is not an fp32 and (with near = 2^-60) every midpoint is an fp64 tie -- bit-exact
    against the oracle's exactly rounded lattice (reading #3)."""
    rng = np.random.default_rng(77 + res + strat)
    n = 4000
    dist = rng.uniform(4200.0, 15500.0, n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = (rng.uniform(-0.45, 0.45, (n, 3)) - dist[:, None] * d).astype(np.float32)
    d = d.astype(np.float32)
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    occ = (rng.random(res**3) < 0.35).astype(np.uint8)
    kw = dict(step=float(np.float32(2.0**-10)), stratified=strat, seed=99)
    ref = O.march(occ, 1, res, roi, o, d, near=float(np.float32(near)), **kw)
    got = gpu_march(N, occ, 1, res, roi, o, d, near_plane=float(np.float32(near)), **kw)
    assert_march_equal(got, ref)
    k = np.round(ref[1].astype(np.float64) / 2.0**-10)
    assert k.min() >= (1 << 22) and k.max() >= (1 << 23) and ref[0][:, 1].sum() > 50000


def test_march_cone_table_overflow_raises(N):
    """a cone lattice longer than the 2^20-entry shared table must not return
    silently truncated samples; the synchronous path reads the device status and raises."""
    rng = np.random.default_rng(3)
    o, d = random_rays(64, rng)
    with pytest.raises(N.NaccError):
        gpu_march(N, np.ones(8**3, np.uint8), 1, 8, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d,
                  step=float(np.float32(1e-6)), cone_angle=float(np.float32(1e-9)),
                  max_step=float(np.float32(1e-6)), near_plane=0.2)


def test_march_edge_cases(N):
    rng = np.random.default_rng(1)
    o, d = random_rays(500, rng)
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    empty = np.zeros(8**3, np.uint8)
    pk, t0, _, _ = gpu_march(N, empty, 1, 8, roi, o, d, step=0.01)  # all-empty grid
    assert pk[:, 1].sum() == 0 and len(t0) == 0 and np.all(pk[:, 0] == 0)
    # all rays miss
    om = o + np.array([10, 10, 10], np.float32)
    pk, t0, _, _ = gpu_march(N, np.ones(8**3, np.uint8), 1, 8, roi, om, d, step=0.01)
    assert pk[:, 1].sum() == 0
    # zero rays
    pk, t0, _, _ = gpu_march(N, np.ones(8**3, np.uint8), 1, 8, roi, o[:0], d[:0], step=0.01)
    assert pk.shape == (0, 2) and len(t0) == 0
    # one-shot with a too-small capacity falls back to the fill path
    full = np.ones(8**3, np.uint8)
    ref = O.march(full, 1, 8, roi, o, d, step=0.01)
    got = gpu_march(N, full, 1, 8, roi, o, d, step=0.01, capacity=17)
    assert_march_equal(got, ref)
    got = gpu_march(N, full, 1, 8, roi, o, d, step=0.01, capacity=len(ref[1]) + 5)
    assert_march_equal(got, ref)
    # long rays spanning many warp iterations (tiny step)
    ref = O.march(full, 1, 8, roi, o[:50], d[:50], step=1e-4)
    assert ref[0][:, 1].max() > 5000
    assert_march_equal(gpu_march(N, full, 1, 8, roi, o[:50], d[:50], step=1e-4), ref)


@pytest.mark.parametrize("levels,res", [(1, 16), (3, 12), (2, 13)])
def test_march_sparse_grid_bounds(N, levels, res):
    """A handful of occupied cells (box corners, level boundaries): the march
    narrows each ray's scan to the box enclosing the occupied cells, which must
    never drop an emitted interval."""
    rng = np.random.default_rng(50 + levels + res)
    o, d = random_rays(4000, rng)
    occ = np.zeros(levels * res**3, np.uint8)
    picks = [0, res - 1, res * res - 1, res**3 - 1, (res // 2) * (1 + res + res * res)]
    for l in range(levels):
        for c in picks:
            occ[l * res**3 + c] = 1
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    step = float(np.float32(0.003))
    ref = O.march(occ, levels, res, roi, o, d, step=step)
    assert ref[0][:, 1].sum() > 100
    assert_march_equal(gpu_march(N, occ, levels, res, roi, o, d, step=step), ref)
    one = np.zeros_like(occ)
    one[(levels - 1) * res**3 + res**3 - 1] = 1  # only the outermost level's last corner cell
    ref = O.march(one, levels, res, roi, o * 3, d, step=step)
    assert_march_equal(gpu_march(N, one, levels, res, roi, o * 3, d, step=step), ref)


@pytest.mark.parametrize("cells_per_step", [0.05, 0.2, 0.37, 0.5, 1.3])
def test_march_fine_mask_stress(N, cells_per_step):
    """Single-level grids take the fine (3-cell-window) segment test: isolated occupied
    cells, cells on the box faces and corners, axis-aligned rays along cell boundaries,
    rays starting inside the box, and steps whose 8-point segments span 0.4 .. 10 cells
    (beyond 3 cells per axis the test falls back to full evaluation).  Bit-exact."""
    R = 32
    rng = np.random.default_rng(int(cells_per_step * 1000))
    occ = (rng.random(R**3) < 0.01).astype(np.uint8)
    idx = np.arange(R)
    for a, b in ((0, 0), (R - 1, R - 1), (0, R - 1), (R - 2, 1)):  # face and corner lines
        occ[a + R * (b + R * idx)] = 1
        occ[idx + R * (a + R * b)] = 1
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    o, d = random_rays(3000, rng)
    # axis-aligned rays exactly on cell boundaries, and origins inside the box
    k = 400
    j = rng.integers(0, R + 1, (k, 2)) / R - 0.5
    ax = rng.integers(0, 3, k)
    for i in range(k):
        oo = np.empty(3)
        oo[ax[i]] = -0.9
        oo[(ax[i] + 1) % 3], oo[(ax[i] + 2) % 3] = j[i]
        dd = np.zeros(3)
        dd[ax[i]] = 1.0
        o[5 + i], d[5 + i] = oo, dd
    o[500:800] = rng.uniform(-0.45, 0.45, (300, 3)).astype(np.float32)
    step = float(np.float32(cells_per_step / R))
    ref = O.march(occ, 1, R, roi, o, d, step=step)
    assert ref[0][:, 1].sum() > 500
    assert_march_equal(gpu_march(N, occ, 1, R, roi, o, d, step=step), ref)


def test_march_deterministic(N):
    rng = np.random.default_rng(2)
    o, d = random_rays(4000, rng)
    occ = (rng.random(16**3) < 0.4).astype(np.uint8)
    a = gpu_march(N, occ, 1, 16, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, step=0.003, stratified=1, seed=9)
    b = gpu_march(N, occ, 1, 16, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, step=0.003, stratified=1, seed=9)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.fixture(scope="module")
def cfg2():
    c = W.cfg2()
    ref = O.march(c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step)
    return c, ref


def test_march_cfg2_full(N, cfg2):
    """CFG2 at full size (2^18 rays, 128^3), every ray compared bit-exactly."""
    c, ref = cfg2
    assert_march_equal(gpu_march(N, c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step), ref)
    # the one-shot (single-pass, look-back) path the bench times
    assert_march_equal(gpu_march(N, c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step,
                                 capacity=len(ref[1]) + 100), ref)


def test_march_cfg3_full(N):
    """CFG3 at full size (640k rays, 4-level cascade, cone steps)."""
    c = W.cfg3()
    ref = O.march(c.occ, 4, 128, c.roi, c.rays_o, c.rays_d, near=c.near, step=c.step, cone_angle=c.cone_angle,
                  max_step=c.max_step)
    got = gpu_march(N, c.occ, 4, 128, c.roi, c.rays_o, c.rays_d, near_plane=c.near, step=c.step,
                    cone_angle=c.cone_angle, max_step=c.max_step)
    assert_march_equal(got, ref)
    got = gpu_march(N, c.occ, 4, 128, c.roi, c.rays_o, c.rays_d, near_plane=c.near, step=c.step,
                    cone_angle=c.cone_angle, max_step=c.max_step, capacity=len(ref[1]))
    assert_march_equal(got, ref)
    assert ref[0][:, 1].mean() > 100
    # the combined estimator's spans on the cascade (the fused kernel in bounds mode): the first t0
    # and the last t1 each ray emits (reading #18), (0, 0) for rays that emit nothing
    pk, t0, t1 = ref[0], ref[1], ref[2]
    has = pk[:, 1] > 0
    tn_ref = np.where(has, t0[np.minimum(pk[:, 0], len(t0) - 1)], 0).astype(np.float32)
    tf_ref = np.where(has, t1[np.minimum(pk[:, 0] + pk[:, 1] - 1, len(t1) - 1)], 0).astype(np.float32)
    tn, tf, alive = gpu_bounds(N, c.occ, 4, 128, c.roi, c.rays_o, c.rays_d, near_plane=c.near, step=c.step,
                               cone_angle=c.cone_angle, max_step=c.max_step)
    assert np.array_equal(tn, tn_ref) and np.array_equal(tf, tf_ref)
    assert alive == int(has.sum())


# ============================================================================ filter
def gpu_filter(N, pk, t0, t1, sig, eps=1e-4):
    import torch

    s = N.PackedSamples(cuda(pk), cuda(t0), cuda(t1), cuda(np.zeros(len(t0), np.int32)))
    f = N.filter_early_stop(s, cuda(sig), eps)
    torch.cuda.synchronize()
    return f.packed_info.cpu().numpy(), f.t0.cpu().numpy(), f.t1.cpu().numpy(), f.ray_id.cpu().numpy()


def check_filter(gpu, ref, margin, L):
    pg, g0, g1, gr = gpu
    pr, r0, r1, rr, _ = ref
    tie = margin < 1e-9 * L
    diff = pg[:, 1] != pr[:, 1]
    assert not np.any(diff & ~tie), f"{np.sum(diff & ~tie)} cuts differ outside the tie band"
    if not diff.any():
        assert np.array_equal(pg, pr) and np.array_equal(g0, r0) and np.array_equal(g1, r1) and np.array_equal(gr, rr)
    return int(tie.sum())


@pytest.mark.parametrize("seed", [0, 1])
def test_filter_ragged(N, seed):
    pk, t0, t1, _, sig, _ = W.ragged_samples(3000, seed=seed, long_rays=(0, 5, 77))
    for eps in (1e-4, 1e-2, 0.0):
        L = -math.log(float(np.float32(eps))) if eps > 0 else math.inf
        ref = O.filter_early_stop(pk, t0, t1, sig, L)
        n_tie = check_filter(gpu_filter(N, pk, t0, t1, sig, eps), ref, ref[4], L)
        assert n_tie == 0


def test_filter_exact_on_near_ties(N):
    """Decisions within rounding of L stay bit-exact: the filter accumulates S_i in the
    definition's sequential order with the same fp64 ops as the oracle (O5), so even an L
    set to the sequential fp64 prefix itself (and 1 ulp off) cuts identically."""
    import ctypes as C

    import torch
    from paper_2305_04966_b200 import _lib as Lb

    rng = np.random.default_rng(31)
    counts = np.array([40, 3, 60, 17, 0, 33] * 20, np.int64)
    pk = np.stack([np.concatenate([[0], np.cumsum(counts)[:-1]]), counts], 1).astype(np.int64)
    n_s = int(counts.sum())
    t0 = np.zeros(n_s, np.float32)
    t1 = np.ones(n_s, np.float32)
    sig = rng.choice(np.float32([0.1, 0.3, 0.7, 0.05]), n_s).astype(np.float32)
    p = sig.astype(np.float64)  # δ = 1 exactly
    S = 0.0
    for i in range(19):  # sequential prefix of the first ray after 19 samples
        S += p[i]
    for L in (S, np.nextafter(S, 0), np.nextafter(S, 10), 2.0, 3.0):
        ref = O.filter_early_stop(pk, t0, t1, sig, L)
        dev = torch.device("cuda")
        d_pk, d_t0, d_t1, d_sig = (torch.from_numpy(x).to(dev) for x in (pk, t0, t1, sig))
        out_pk = torch.empty_like(d_pk)
        o0, o1 = torch.empty_like(d_t0), torch.empty_like(d_t1)
        orid = torch.empty(n_s, dtype=torch.int32, device=dev)
        tot = torch.empty(1, dtype=torch.int64, device=dev)
        lib = Lb.lib()
        ws = torch.empty(lib.nacc_filter_workspace_bytes(len(pk)), dtype=torch.uint8, device=dev)
        ptr = lambda x: C.c_void_p(x.data_ptr())
        st = lib.nacc_filter_early_stop(ptr(d_pk), len(pk), ptr(d_t0), ptr(d_t1), ptr(d_sig), n_s, float(L),
                                        ptr(out_pk), ptr(o0), ptr(o1), ptr(orid), n_s, ptr(tot), ptr(ws), ws.numel(),
                                        None)
        assert st == 0
        torch.cuda.synchronize()
        assert np.array_equal(out_pk.cpu().numpy(), ref[0]), L
        assert int(tot.item()) == len(ref[1])


def test_filter_cfg2_full(N, cfg2):
    c, (pk, t0, t1, rid) = cfg2
    sig, _ = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
    ref = O.filter_early_stop(pk, t0, t1, sig, L_EPS)
    check_filter(gpu_filter(N, pk, t0, t1, sig), ref, ref[4], L_EPS)
    assert len(ref[1]) * 2 < len(t0)  # the filter removes most samples


# ============================================================================ render
def ray_ids(pk):
    return np.repeat(np.arange(len(pk), dtype=np.int32), pk[:, 1])


def gpu_render(N, pk, t0, t1, sig, rgb, g_color, g_opacity, g_depth, eps=None, flat=True):
    import torch

    rid = cuda(ray_ids(pk)) if flat else cuda(np.zeros(0, np.int32))
    s = N.PackedSamples(cuda(pk), cuda(t0), cuda(t1), rid)
    sg = cuda(sig).requires_grad_()
    cg = cuda(rgb).requires_grad_()
    color, opacity, depth = N.rendering(s, sg, cg, eps=eps)
    loss = (color * cuda(g_color)).sum()
    if g_opacity is not None:  # None: opacity / depth unused -> NULL gradients (the colour-only backward)
        loss = loss + (opacity * cuda(g_opacity)).sum() + (depth * cuda(g_depth)).sum()
    loss.backward()
    torch.cuda.synchronize()
    return (color.detach().cpu().numpy(), opacity.detach().cpu().numpy(), depth.detach().cpu().numpy(),
            sg.grad.cpu().numpy(), cg.grad.cpu().numpy())


def close_rel(got, ref, rel=1e-4, floor=1e-6):
    return np.abs(got - ref) <= rel * np.abs(ref) + floor


def grad_ok(got, ref, pk, comps=1):
    ref = ref.reshape(len(ref), -1)
    got = got.reshape(len(got), -1)
    ray_max = np.zeros(len(ref))
    for (s, c) in pk:
        if c:
            ray_max[s : s + c] = np.abs(ref[s : s + c]).max()
    return np.abs(got - ref) <= 1e-3 * (np.abs(ref) + 1e-3 * ray_max[:, None])


def run_render_parity(N, pk, t0, t1, sig, rgb, seed, eps=None, flat=True, color_only=False):
    rng = np.random.default_rng(seed)
    n = len(pk)
    gC, gO, gD = rng.normal(size=(n, 3)).astype(np.float32), rng.normal(size=n).astype(np.float32), \
        rng.normal(size=n).astype(np.float32)
    if color_only:  # a colour loss only: the backward gets NULL opacity / depth gradients
        gO, gD = np.zeros(n, np.float32), np.zeros(n, np.float32)
    L = math.inf if eps is None else -math.log(float(np.float32(eps)))
    got = gpu_render(N, pk, t0, t1, sig, rgb, gC, None if color_only else gO, None if color_only else gD, eps, flat)
    ref = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=L)
    gs, grgb = O.render_bwd(pk, t0, t1, sig, rgb, gC, gO, gD, neg_log_eps=L)
    ok_rays = np.ones(n, bool)
    if eps is not None:  # rays with an early-stop decision in the tie band are compared leniently
        _, margin = O.filter_counts(pk, t0, t1, sig, L)
        ok_rays = margin >= 1e-9 * L
    assert np.all(close_rel(got[0], ref["color"])[ok_rays])
    assert np.all(close_rel(got[1], ref["opacity"])[ok_rays])
    assert np.all(close_rel(got[2], ref["depth"])[ok_rays])
    samp_ok = np.repeat(ok_rays, pk[:, 1])
    assert np.all(grad_ok(got[3], gs, pk)[samp_ok])
    assert np.all(grad_ok(got[4], grgb, pk)[samp_ok])


@pytest.mark.parametrize("eps", [None, 1e-4])
@pytest.mark.parametrize("flat", [True, False])
def test_render_ragged(N, eps, flat):
    """flat = the ray-aligned-tile kernels (ray_id given); False = one warp per ray"""
    pk, t0, t1, _, sig, rgb = W.ragged_samples(2000, seed=3, long_rays=(0, 9, 1500, 1999), long_count=5000)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=4, eps=eps, flat=flat)


@pytest.mark.parametrize("eps", [None, 1e-4])
def test_render_color_only_backward(N, eps):
    """colour loss only (opacity / depth unused): the backward skips the per-ray constants kernel
    and reads g_C and the forward's colour sums directly (render.cu kColorOnly)"""
    pk, t0, t1, _, sig, rgb = W.ragged_samples(2000, seed=23, long_rays=(0, 9, 1500, 1999), long_count=5000)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=24, eps=eps, color_only=True)


def test_render_flat_unaligned(N):
    """odd offsets take the scalar (non-vector) path of the flat kernels"""
    pk, t0, t1, _, sig, rgb = W.ragged_samples(500, seed=13)
    pk2 = pk.copy()
    pk2[:, 0] += 1
    pad = lambda a: np.concatenate([np.zeros((1,) + a.shape[1:], a.dtype), a])
    import torch

    s = N.PackedSamples(cuda(pk2), cuda(pad(t0))[1:], cuda(pad(t1))[1:], cuda(pad(ray_ids(pk)))[1:])
    # the binding passes the (unaligned) views straight through
    sg = cuda(pad(sig))[1:]
    cg = cuda(pad(rgb))[1:]
    s = N.PackedSamples(cuda(pk), s.t0, s.t1, s.ray_id)
    color, opacity, depth = N.rendering(s, sg, cg)
    ref = O.render_fwd(pk, t0, t1, sig, rgb)
    assert np.all(close_rel(color.cpu().numpy(), ref["color"]))
    assert np.all(close_rel(depth.cpu().numpy(), ref["depth"]))
    torch.cuda.synchronize()


def test_render_degenerate(N):
    # zero-sample rays, σ ≡ 0 rays, one opaque interval
    pk = np.array([[0, 0], [0, 3], [3, 0], [3, 1]], np.int64)
    t0 = np.array([0.0, 0.1, 0.2, 1.0], np.float32)
    t1 = np.array([0.1, 0.2, 0.3, 1.5], np.float32)
    sig = np.array([0.0, 0.0, 0.0, 1e4], np.float32)
    rgb = np.full((4, 3), 0.5, np.float32)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=5)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=5, eps=1e-4)


@pytest.fixture(scope="module")
def cfg2_filtered(cfg2):
    c, (pk, t0, t1, rid) = cfg2
    sig, _ = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
    pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, L_EPS)
    s2, rgb2 = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, a0, a1, r2)
    return pk2, a0, a1, r2, s2, rgb2


def test_render_cfg2_full(N, cfg2_filtered):
    """CFG2 full size, post-filter samples, every ray."""
    pk2, a0, a1, r2, s2, rgb2 = cfg2_filtered
    run_render_parity(N, pk2, a0, a1, s2, rgb2, seed=6, eps=1e-4)


def test_render_cfg1(N):
    c = W.cfg1()
    pk, t0, t1, rid = O.march(c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step)
    sig, rgb = W.field_at_intervals(W.sphere_sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=7)
    run_render_parity(N, pk, t0, t1, sig, rgb, seed=7, eps=1e-4)


def test_weights_and_accumulate(N):
    import torch

    pk, t0, t1, _, sig, rgb = W.ragged_samples(1500, seed=8, long_rays=(3,))
    # flat = ray_id given (the flat-tile forward); else an empty ray_id (one warp per ray)
    for eps, flat in ((None, True), (1e-4, True), (None, False), (1e-4, False)):
        L = math.inf if eps is None else -math.log(float(np.float32(eps)))
        rid = cuda(ray_ids(pk)) if flat else cuda(np.zeros(0, np.int32))
        s = N.PackedSamples(cuda(pk), cuda(t0), cuda(t1), rid)
        sg = cuda(sig).requires_grad_()
        w, T, a = N.render_weights(s, sg, eps=eps)
        ref = O.render_fwd(pk, t0, t1, sig, None, neg_log_eps=L)
        _, margin = O.filter_counts(pk, t0, t1, sig, L)
        ok = np.repeat(margin >= 1e-9 * L, pk[:, 1])
        assert np.all((np.abs(w.detach().cpu().numpy() - ref["weights"]) <= 1e-5)[ok])
        assert np.all(np.abs(T.detach().cpu().numpy() - ref["trans"]) <= 1e-5)
        assert np.all(np.abs(a.detach().cpu().numpy() - ref["alphas"]) <= 1e-5)
        rng = np.random.default_rng(9)
        gw, gT = rng.normal(size=len(t0)).astype(np.float32), rng.normal(size=len(t0)).astype(np.float32)
        (w * cuda(gw)).sum().add_((T * cuda(gT)).sum()).backward()
        gs = O.weights_bwd(pk, t0, t1, sig, gw, gT, neg_log_eps=L)
        assert np.all(grad_ok(sg.grad.cpu().numpy(), gs, pk)[ok])
    # accumulate fwd/bwd with C = 1 (opacity), 3 (rgb) and 5, flat (ray_id) and one warp per ray
    w = torch.rand(len(t0), device="cuda", requires_grad=True)
    s_flat = N.PackedSamples(cuda(pk), cuda(t0), cuda(t1), cuda(ray_ids(pk)))
    for C_, s in [(c, sx) for sx in (s, s_flat) for c in (None, 2, 3, 4, 5)]:
        vals = None if C_ is None else torch.rand(len(t0), C_, device="cuda", requires_grad=True)
        out = N.accumulate_along_rays(s, w, vals)
        g = torch.randn_like(out)
        out.backward(g)
        wn = w.detach().cpu().numpy()
        vn = None if vals is None else vals.detach().cpu().numpy()
        ref = O.accumulate(pk, wn, vn, C_=1)
        assert np.all(close_rel(out.detach().cpu().numpy(), ref, 1e-5, 1e-6))
        gw_ref, gv_ref = O.accumulate_bwd(pk, wn, vn, g.cpu().numpy())
        assert np.all(close_rel(w.grad.cpu().numpy(), gw_ref, 1e-5, 1e-6))
        if vals is not None:
            assert np.all(close_rel(vals.grad.cpu().numpy(), gv_ref, 1e-6, 1e-7))
        w.grad = None


@pytest.mark.parametrize("eps", [None, 1e-4])
@pytest.mark.parametrize("flat", [True, False])
def test_weights_alpha(N, eps, flat):
    """Alpha compositing (readings #16-#17) vs the oracle: ragged rays incl.
    5000-sample ones, α with exact 0s and 1s (opaque samples), early stop."""
    import torch

    pk, _, _, _, _, _ = W.ragged_samples(1500, seed=21, long_rays=(2, 700), long_count=5000)
    n_s = int(pk[:, 1].sum())
    rng = np.random.default_rng(22)
    a = rng.choice([0.0, 1.0, 0.02, 0.3], n_s, p=[0.3, 0.01, 0.5, 0.19]).astype(np.float32)
    a *= rng.uniform(0.5, 1.0, n_s).astype(np.float32) ** (a < 1)
    L = math.inf if eps is None else -math.log(float(np.float32(eps)))
    # flat: ray_id given (the flat-tile forward); else an empty ray_id (one warp per ray)
    s = N.PackedSamples(cuda(pk), cuda(np.zeros(n_s, np.float32)), cuda(np.zeros(n_s, np.float32)),
                        cuda(ray_ids(pk)) if flat else cuda(np.zeros(0, np.int32)))
    ag = cuda(a).requires_grad_()
    w, T = N.render_weights_alpha(s, ag, eps=eps)
    w_ref, T_ref = O.weights_alpha_fwd(pk, a, L)
    # decisions within 1e-9 relative of ε_T are a tie band (product order differs)
    eps_T = math.exp(-L)
    tie = np.zeros(len(pk), bool)
    if eps is not None:
        near = np.abs(T_ref - eps_T) <= 1e-9 * eps_T
        tie = np.add.reduceat(near.astype(np.int64), np.minimum(pk[:, 0], max(n_s - 1, 0))) > 0
        tie &= pk[:, 1] > 0
    ok = np.repeat(~tie, pk[:, 1])
    assert np.all((np.abs(w.detach().cpu().numpy() - w_ref) <= 1e-5)[ok])
    assert np.all(np.abs(T.detach().cpu().numpy() - T_ref) <= 1e-5)
    gw, gT = rng.normal(size=n_s).astype(np.float32), rng.normal(size=n_s).astype(np.float32)
    (w * cuda(gw)).sum().add_((T * cuda(gT)).sum()).backward()
    ga = O.weights_alpha_bwd(pk, a, gw, gT, neg_log_eps=L)
    assert np.all(grad_ok(ag.grad.cpu().numpy(), ga, pk)[ok])


# ============================================================================ resample
def check_resample(s_gpu, s_ref, F_ref, e, n_out, stratified=False, seed=0):
    n = len(s_gpu)
    for r in range(n):
        Fh = F_ref[r]
        back = np.interp(s_gpu[r].astype(np.float64), e[r].astype(np.float64), Fh)
        slope = np.diff(Fh) / np.maximum(np.diff(e[r].astype(np.float64)), 1e-30)
        jj = np.clip(np.searchsorted(e[r], s_gpu[r], side="right") - 1, 0, len(slope) - 1)
        steep = np.maximum(slope[jj], slope[np.maximum(jj - 1, 0)])  # an edge on a bin boundary sees both
        ulp = np.spacing(np.abs(s_gpu[r]).astype(np.float32)).astype(np.float64)
        if not stratified:
            u = np.arange(n_out + 1) / n_out
            # 1e-6 plus the fp32 rounding of the output edge (slope x 1 ulp)
            assert np.all(np.abs(back - u) <= 1e-6 + steep * ulp), r
        assert np.all(np.diff(s_gpu[r]) >= 0)
        j = np.clip(np.searchsorted(e[r], s_ref[r], side="right") - 1, 0, len(slope) - 1)
        steep = slope[j] >= 1e-2
        assert np.all(np.abs(s_gpu[r] - s_ref[r])[steep] <= 1e-5)


def test_resample_cfg4_full(N):
    """CFG4: 2^16 rays, 256 -> 96 -> 48 (lindisp, t_n = 0.2, t_f = 1000)."""
    import torch

    p = W.cfg4()
    n = len(p.rays_o)
    e0 = p.s_edges
    tm = W.lindisp(0.5 * (e0[:, :-1].astype(np.float64) + e0[:, 1:]), p.t_near, p.t_far)
    x = p.rays_o[:, None, :].astype(np.float64) + tm[..., None] * p.rays_d[:, None, :]
    sig1, _ = p.scene.sigma_rgb(x)
    sig1 = sig1.astype(np.float32)
    s1_gpu, t1_gpu = N.importance_sample(cuda(e0), 96, sigma=cuda(sig1), map_kind=N.MAP_LINDISP, t_near=p.t_near,
                                         t_far=p.t_far)
    s1_ref, t1_ref = O.importance_sample(e0, 96, sigma=sig1, map_kind=1, t_near=p.t_near, t_far=p.t_far)
    F1 = O.importance_cdf(e0, sigma=sig1, map_kind=1, t_near=p.t_near, t_far=p.t_far)
    s1g = s1_gpu.cpu().numpy()
    pick = np.random.default_rng(0).choice(n, 4096, replace=False)
    check_resample(s1g[pick], s1_ref[pick], F1[pick], e0[pick], 96)
    tg = t1_gpu.cpu().numpy().astype(np.float64)  # t_out = Φ(s_out): check it in s-space (Φ is steep near s = 1)
    s_back = (1.0 / tg - 1.0 / p.t_near) / (1.0 / p.t_far - 1.0 / p.t_near)
    assert np.abs(s_back - s1g).max() <= 1e-6
    # round 2 from the oracle's round-1 edges (inputs never come from the CUDA path)
    e1 = s1_ref.astype(np.float32)
    tm2 = W.lindisp(0.5 * (e1[:, :-1].astype(np.float64) + e1[:, 1:]), p.t_near, p.t_far)
    x2 = p.rays_o[:, None, :].astype(np.float64) + tm2[..., None] * p.rays_d[:, None, :]
    sig2 = p.scene.sigma_rgb(x2)[0].astype(np.float32)
    s2_gpu, _ = N.importance_sample(cuda(e1), 48, sigma=cuda(sig2), map_kind=N.MAP_LINDISP, t_near=p.t_near,
                                    t_far=p.t_far)
    s2_ref, _ = O.importance_sample(e1, 48, sigma=sig2, map_kind=1, t_near=p.t_near, t_far=p.t_far)
    F2 = O.importance_cdf(e1, sigma=sig2, map_kind=1, t_near=p.t_near, t_far=p.t_far)
    check_resample(s2_gpu.cpu().numpy()[pick], s2_ref[pick], F2[pick], e1[pick], 48)
    torch.cuda.synchronize()


def test_resample_cdf_input_stratified_and_degenerate(N):
    rng = np.random.default_rng(11)
    n, m = 700, 40
    e = np.sort(rng.uniform(0, 1, (n, m + 1)), axis=1).astype(np.float32)
    e[:, 0], e[:, -1] = 0, 1
    w = np.where(rng.random((n, m)) < 0.4, 0, rng.uniform(0, 1, (n, m)))
    w[:5] = 0.0  # zero-mass rays -> uniform edges
    cdf = np.concatenate([np.zeros((n, 1)), np.cumsum(w, 1)], 1).astype(np.float32)
    sg, _ = N.importance_sample(cuda(e), 33, cdf=cuda(cdf), map_kind=N.MAP_IDENTITY, t_near=1.0, t_far=5.0)
    sr, _ = O.importance_sample(e, 33, cdf=cdf, map_kind=0, t_near=1.0, t_far=5.0)
    F = O.importance_cdf(e, cdf=cdf, map_kind=0, t_near=1.0, t_far=5.0)
    check_resample(sg.cpu().numpy(), sr, F, e, 33)
    sig = rng.uniform(0, 20, (n, m)).astype(np.float32)
    sg, _ = N.importance_sample(cuda(e), 17, sigma=cuda(sig), map_kind=N.MAP_LINDISP, stratified=True, seed=5)
    sr, _ = O.importance_sample(e, 17, sigma=sig, map_kind=1, stratified=1, seed=5)
    F = O.importance_cdf(e, sigma=sig, map_kind=1)
    check_resample(sg.cpu().numpy(), sr, F, e, 17, stratified=True)


def test_resample_unbounded_lindisp(N):
    """Φ = lindisp with t_f = inf (1/t = (1 - s)/t_n): t grows without bound as s -> 1;
    the kernel's reciprocals must follow the oracle out to t ~ 1e6."""
    rng = np.random.default_rng(21)
    n, m = 500, 64
    e = np.sort(rng.uniform(0, 0.999999, (n, m + 1)), axis=1).astype(np.float32)
    e[:, 0] = 0
    sig = rng.uniform(0, 3, (n, m)).astype(np.float32)
    sg, tg = N.importance_sample(cuda(e), 24, sigma=cuda(sig), map_kind=N.MAP_LINDISP, t_near=0.5,
                                 t_far=math.inf)
    sr, tr = O.importance_sample(e, 24, sigma=sig, map_kind=1, t_near=0.5, t_far=math.inf)
    F = O.importance_cdf(e, sigma=sig, map_kind=1, t_near=0.5, t_far=math.inf)
    check_resample(sg.cpu().numpy(), sr, F, e, 24)
    tg = tg.cpu().numpy().astype(np.float64)
    s32 = sg.cpu().numpy()
    t_of_s = 1.0 / ((1.0 - s32.astype(np.float64)) / 0.5)  # Φ of the kernel's own (rounded) s
    # the kernel maps its unrounded s: allow dΦ/ds = t^2 / t_n times one fp32 ulp of s
    ulp = np.spacing(np.abs(s32)).astype(np.float64)
    assert np.all(np.abs(tg - t_of_s) <= 1e-6 * t_of_s + t_of_s**2 / 0.5 * ulp)


@pytest.mark.parametrize("map_kind", [0, 1])
def test_resample_far_mass(N, map_kind):
    """Mass in the far bins (s -> 1, where 1/t is small for lindisp): the kernel's fp32 interval
    lengths (reading #29) must not lose it to cancellation; n_in 256 / 96 / 40 (8, 3, 2 edges per
    lane) and t_out against Φ(s_out)."""
    rng = np.random.default_rng(31)
    for m, n_out in ((256, 96), (96, 48), (40, 17)):
        n = 600
        e = np.sort(rng.uniform(0, 1, (n, m + 1)), axis=1).astype(np.float32)
        e[:, 0], e[:, -1] = 0, 1
        mid = 0.5 * (e[:, :-1] + e[:, 1:])
        sig = np.where(mid > 0.85, rng.uniform(0.5, 40, (n, m)), rng.uniform(0, 0.02, (n, m))).astype(np.float32)
        tn, tf = 0.2, 1000.0
        # rays 0..99: mass only in a middle bin and in a last bin that starts at s = 1 - 1e-4, where
        # 1/t_n + s (1/t_f - 1/t_n) would cancel (its fp32 Δt is off by ~3e-4 there; ~4e-6 in F)
        e[:100, -2] = np.float32(1 - 1e-4)
        e[:100, :-1] = np.minimum(e[:100, :-1], np.float32(1 - 1e-4))
        t64 = 1.0 / ((1.0 - e[:100].astype(np.float64)) / tn + e[:100].astype(np.float64) / tf)
        dt = np.maximum(np.diff(t64, axis=1), 1e-12)
        sig[:100] = 0.0
        sig[:100, m // 2] = (0.7 / dt[:, m // 2]).astype(np.float32)
        sig[:100, -1] = (0.7 / dt[:, -1]).astype(np.float32)
        sg, tg = N.importance_sample(cuda(e), n_out, sigma=cuda(sig), map_kind=map_kind, t_near=tn, t_far=tf)
        sr, _ = O.importance_sample(e, n_out, sigma=sig, map_kind=map_kind, t_near=tn, t_far=tf)
        F = O.importance_cdf(e, sigma=sig, map_kind=map_kind, t_near=tn, t_far=tf)
        sg, tg = sg.cpu().numpy(), tg.cpu().numpy().astype(np.float64)
        check_resample(sg, sr, F, e, n_out)
        s64 = sg.astype(np.float64)
        t_ref = 1.0 / ((1.0 - s64) / tn + s64 / tf) if map_kind == 1 else tn + s64 * (tf - tn)
        assert np.all(np.abs(tg - t_ref) <= 4e-7 * t_ref + 1e-6)


# ============================================================================ combined estimator
def gpu_bounds(N, occ, levels, res, roi, o, d, **kw):
    import torch

    spec = N.GridSpec(roi=roi, res=res, levels=levels)
    bits = N.prepare_bits(spec, cuda(W.pack_bits(occ).view(np.int32)))
    tn, tf, alive = N.occgrid_ray_bounds(cuda(o), cuda(d), spec, bits, N.MarchParams(**kw))
    torch.cuda.synchronize()
    return tn.cpu().numpy(), tf.cpu().numpy(), int(alive.item())


def test_ray_bounds_bit_exact(N, cfg2):
    """Readings #18: the span equals the first t0 / last t1 the march emits, bit-exactly."""
    c, _ = cfg2
    tn_r, tf_r = O.ray_bounds(c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step)
    tn, tf, alive = gpu_bounds(N, c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step)
    assert np.array_equal(tn, tn_r) and np.array_equal(tf, tf_r)
    assert alive == int((tf_r > tn_r).sum()) > 1000
    rng = np.random.default_rng(41)
    o, d = random_rays(3000, rng)
    roi = (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    for levels, res, cone in ((1, 16, 0), (3, 8, 1), (2, 13, 0)):
        occ = (rng.random(levels * res**3) < 0.1).astype(np.uint8)
        kw = dict(step=float(np.float32(0.005)))
        if cone:
            kw.update(cone_angle=float(np.float32(1 / 128)), max_step=float(np.float32(0.05)), near=0.02)
        ref = O.ray_bounds(occ, levels, res, roi, o, d, **kw)
        if "near" in kw:
            kw["near_plane"] = kw.pop("near")
        got = gpu_bounds(N, occ, levels, res, roi, o, d, **kw)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    tn, tf, alive = gpu_bounds(N, np.zeros(8**3, np.uint8), 1, 8, roi, o, d, step=0.01)
    assert alive == 0 and not tn.any() and not tf.any()


def test_combined_estimator_cfg2(N, cfg2):
    """Readings #18-#19 on CFG2 rays: grid spans, then one proposal round
    (64 -> 32 edges, identity map inside each span) vs the oracle; culled
    rays get uniform edges at t_near."""
    import torch

    c, _ = cfg2
    sub = np.random.default_rng(42).choice(len(c.rays_o), 3000, replace=False)
    o, d = c.rays_o[sub], c.rays_d[sub]
    tn, tf = O.ray_bounds(c.occ, 1, 128, c.roi, o, d, step=c.step)
    n, m = len(o), 64
    e0 = np.tile(np.linspace(0, 1, m + 1, dtype=np.float32), (n, 1))
    tm = tn[:, None].astype(np.float64) + 0.5 * (e0[:, :-1] + e0[:, 1:]) * (tf - tn)[:, None]
    x = o[:, None, :].astype(np.float64) + tm[..., None] * d[:, None, :]
    sig = c.scene.sigma_rgb(x.reshape(-1, 3))[0].reshape(n, m).astype(np.float32)
    sg, tg = N.importance_sample(cuda(e0), 32, sigma=cuda(sig), map_kind=N.MAP_IDENTITY, t_near=cuda(tn),
                                 t_far=cuda(tf))
    sr, trr = O.importance_sample_ranged(e0, 32, tn, tf, sigma=sig, map_kind=0)
    torch.cuda.synchronize()
    sg, tg = sg.cpu().numpy(), tg.cpu().numpy()
    live = tf > tn
    assert live.sum() > 1000 and (~live).sum() > 100
    assert np.array_equal(sg[~live], sr[~live].astype(np.float32)) and np.all(tg[~live] == tn[~live, None])
    idx = np.nonzero(live)[0]
    F = np.stack([O.importance_cdf(e0[r:r + 1], sigma=sig[r:r + 1], map_kind=0, t_near=float(tn[r]),
                                   t_far=float(tf[r]))[0] for r in idx])
    check_resample(sg[idx], sr[idx], F, e0[idx], 32)
    # t_out = Φ_r(s_out) on each ray's own span
    assert np.allclose(tg[idx], tn[idx, None] + sg[idx].astype(np.float64) * (tf - tn)[idx, None], rtol=2e-7,
                       atol=1e-6)


# ============================================================================ grid update
def test_occgrid_points_bit_exact(N):
    import torch

    for levels, res, roi in ((1, 128, (0, 0, 0, 1, 1, 1)), (4, 32, (-1, -1, -1, 1, 1, 1)), (2, 7, (-0.3, 0, 1, 0.9, 2, 1.5))):
        g = N.OccupancyGrid(N.GridSpec(roi=roi, res=res, levels=levels), seed=77)
        for jitter in (0, 1):
            got = g.points(5, bool(jitter)).cpu().numpy()
            ref = O.occgrid_points(levels, res, roi, seed=77, step=5, jitter=jitter)
            assert np.array_equal(got, ref)
        nc = levels * res**3
        got = g.points(9, True, nc // 3, nc // 2).cpu().numpy()
        ref = O.occgrid_points(levels, res, roi, seed=77, step=9, jitter=1, cell_begin=nc // 3, cell_count=nc // 2)
        assert np.array_equal(got, ref)
    torch.cuda.synchronize()


@pytest.mark.parametrize("rule,thresh_rule", [(0, 0), (1, 0), (0, 1)])
def test_occgrid_update_bit_exact(N, rule, thresh_rule):
    import torch

    levels, res = 2, 64
    rng = np.random.default_rng(12 + rule + 2 * thresh_rule)
    dens = rng.uniform(0, 0.05, levels * res**3).astype(np.float32)
    g = N.OccupancyGrid(N.GridSpec(roi=(-1, -1, -1, 1, 1, 1), res=res, levels=levels), decay=0.95, threshold=0.01,
                        rule=rule, thresh_rule=thresh_rule)
    g.density.copy_(cuda(dens))
    ref_d = dens.copy()
    for it in range(4):
        fresh = np.where(rng.random(dens.size) < 0.1, rng.uniform(0, 0.5, dens.size), 0).astype(np.float32)
        g.update(cuda(fresh))
        ref_d, ref_b, mean = O.occgrid_update(levels, res, (-1, -1, -1, 1, 1, 1), ref_d, fresh, rule=rule, decay=0.95,
                                              threshold=0.01, thresh_rule=thresh_rule)
        got_d = g.density.cpu().numpy()
        assert np.array_equal(got_d, ref_d)
        got_b = np.unpackbits(g.bits.cpu().numpy().view(np.uint8), bitorder="little")[: dens.size]
        tau = min(0.01, mean) if thresh_rule else 0.01
        tie = np.abs(ref_d.astype(np.float64) - tau) < 1e-12 * max(tau, 1e-30)
        assert np.array_equal(got_b[~tie], ref_b[~tie])
        assert abs(g.mean.item() - mean) <= 1e-12 * max(mean, 1e-30)
    torch.cuda.synchronize()


def test_update_every_n_steps_single_rank(N):
    import torch

    spec = N.GridSpec(roi=(0, 0, 0, 1, 1, 1), res=32)
    g = N.OccupancyGrid(spec, seed=3)
    box = lambda x: ((x < 0.5).all(dim=1).float() * 0.3)  # ConstantBox covering 1/8
    for step in range(33):
        g.update_every_n_steps(step, box, n=16, jitter=False)
    torch.cuda.synchronize()
    bits = np.unpackbits(g.bits.cpu().numpy().view(np.uint8), bitorder="little")[: spec.n_cells]
    assert bits.mean() == 0.125  # 3 updates with γ = 0.95: 0.3·(1-0.95^3) > 0.01


def test_dynamic_grid_times_and_max_merge(N):
    """Reading #20: per-cell timestamps bit-exact vs the oracle (both sides run
    Philox4x32-10); the MAX merge of draws and the update on the merged values
    bit-exact; update_every_n_steps(time_draws=K) reproduces the oracle grid."""
    import torch

    levels, R = 2, 16
    roi = (0, 0, 0, 1, 1, 1)
    spec = N.GridSpec(roi=roi, res=R, levels=levels)
    g = N.OccupancyGrid(spec, seed=11, decay=0.9, threshold=0.1)  # one update: occ = 0.1 σ
    for draw in (0, 5):
        t_gpu = g.times(step=32, draw=draw).cpu().numpy()
        assert np.array_equal(t_gpu, O.occgrid_times(levels, R, roi, 11, 32, draw))
    part = g.times(step=32, draw=1, cell_begin=1000, cell_count=777).cpu().numpy()
    assert np.array_equal(part, O.occgrid_times(levels, R, roi, 11, 32, 1, cell_begin=1000, cell_count=777))
    rng = np.random.default_rng(12)
    a, b = rng.uniform(0, 1, 1001).astype(np.float32), rng.uniform(0, 1, 1001).astype(np.float32)
    da = cuda(a.copy())
    N.max_merge(da, cuda(b))
    assert np.array_equal(da.cpu().numpy(), np.maximum(a, b))
    # a moving sphere, K = 6 draws, one update at step 0.  The caller's field is not the method:
    # record exactly what it returned for each draw (and where/when it was asked), so the oracle
    # merges and updates the identical values and the comparison is bit-exact.
    K = 6
    seen = []

    def sphere(x, t):
        c = torch.stack([0.3 + 0.4 * t, torch.full_like(t, 0.5), torch.full_like(t, 0.5)], 1)
        v = ((x - c).norm(dim=1) < 0.2).float() * 3.0
        seen.append((x.cpu().numpy().copy(), t.cpu().numpy().copy(), v.cpu().numpy().copy()))
        return v

    g.update_every_n_steps(0, sphere, n=16, jitter=True, time_draws=K)
    torch.cuda.synchronize()
    assert len(seen) == K
    xyz = O.occgrid_points(levels, R, roi, 11, 0, 1)
    fresh = None
    for j, (x, t, v) in enumerate(seen):
        assert np.array_equal(x, xyz)  # points: bit-exact (Philox jitter on both sides)
        assert np.array_equal(t, O.occgrid_times(levels, R, roi, 11, 0, j))
        fresh = v if fresh is None else np.maximum(fresh, v)  # MAX over time, reading #20
    dens, bits, _ = O.occgrid_update(levels, R, roi, np.zeros(spec.n_cells, np.float32), fresh, decay=0.9,
                                     threshold=0.1)
    got = np.unpackbits(g.bits.cpu().numpy().view(np.uint8), bitorder="little")[: spec.n_cells]
    assert got.sum() > 50
    assert np.array_equal(got, bits)
    assert np.array_equal(g.density.cpu().numpy(), dens)


def test_pdf_loss(N):
    """Reading #21: proposal-supervision loss and its backward vs the oracle on
    CFG4-shaped histograms (48 final vs 96 / 256 proposal bins) incl. shared
    edges and violated bounds."""
    import torch

    rng = np.random.default_rng(61)
    n = 4096
    for nf, np_ in ((48, 96), (48, 256), (32, 8)):
        t = np.sort(rng.uniform(0, 1, (n, nf + 1)), axis=1).astype(np.float32)
        t[:, 0], t[:, -1] = 0, 1
        w = (rng.dirichlet(np.ones(nf), n) * rng.uniform(0.3, 1, (n, 1))).astype(np.float32)
        th = np.sort(rng.uniform(0, 1, (n, np_ + 1)), axis=1).astype(np.float32)
        th[:, 0], th[:, -1] = 0, 1
        k = min(nf, np_) // 2  # rows 0..9 share k final edges (boundary ties), still ascending
        th[:10] = np.sort(np.concatenate([t[:10, 1 : k + 1], rng.uniform(0, 1, (10, np_ + 1 - k))], 1), axis=1)
        th[:10, 0], th[:10, -1] = 0, 1
        wh = (rng.dirichlet(np.ones(np_), n) * rng.uniform(0.2, 1, (n, 1))).astype(np.float32)
        whg = cuda(wh).requires_grad_()
        loss = N.pdf_loss(cuda(t), cuda(w), cuda(th), whg)
        g = rng.normal(size=n).astype(np.float32)
        (loss * cuda(g)).sum().backward()
        torch.cuda.synchronize()
        ref = O.pdf_loss(t, w, th, wh)
        gref = O.pdf_loss_bwd(t, w, th, wh, g)
        assert np.all(np.abs(loss.detach().cpu().numpy() - ref) <= 1e-4 * np.abs(ref) + 1e-7)
        ga = whg.grad.cpu().numpy()
        scale = np.abs(gref).max(axis=1, keepdims=True) + 1e-6
        assert np.all(np.abs(ga - gref) <= 1e-4 * np.abs(gref) + 1e-5 * scale)
        assert (ref > 0).mean() > 0.5
