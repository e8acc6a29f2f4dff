"""Pins for the combined estimator's oracle pieces (
P:120-122; readings #18-#19): the per-ray span of the grid march and
the proposal resampler restricted to per-ray spans.  Reference values come
from the already pinned march and scalar resampler, closed forms and
invariants."""
import numpy as np

import oracle as O
import workloads as W


def random_rays(n, rng):
    o = 0.5 + rng.normal(size=(n, 3)) * 1.2
    d = 0.5 + rng.uniform(-0.3, 0.3, (n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o.astype(np.float32), d.astype(np.float32)


def test_bounds_are_the_span_of_the_march():
    """t_near / t_far = first t0 / last t1 of what march() emits; culled = none emitted."""
    rng = np.random.default_rng(1)
    o, d = random_rays(600, rng)
    for levels, res, cone in ((1, 16, 0.0), (3, 8, float(np.float32(1 / 64)))):
        occ = (rng.random(levels * res**3) < 0.08).astype(np.uint8)
        kw = dict(step=float(np.float32(0.004)))
        if cone:
            kw.update(cone_angle=cone, max_step=0.05, near=0.05)
        pk, t0, t1, _ = O.march(occ, levels, res, (0, 0, 0, 1, 1, 1), o, d, **kw)
        tn, tf = O.ray_bounds(occ, levels, res, (0, 0, 0, 1, 1, 1), o, d, **kw)
        for r, (s, c) in enumerate(pk):
            if c:
                assert tn[r] == t0[s] and tf[r] == t1[s + c - 1]
            else:
                assert tn[r] == 0 and tf[r] == 0
        assert (pk[:, 1] > 0).sum() > 50 and (pk[:, 1] == 0).sum() > 50


def test_empty_grid_culls_every_ray():
    rng = np.random.default_rng(2)
    o, d = random_rays(200, rng)
    tn, tf = O.ray_bounds(np.zeros(8**3, np.uint8), 1, 8, (0, 0, 0, 1, 1, 1), o, d, step=0.01)
    assert not tn.any() and not tf.any()


def test_full_grid_bounds_closed_form():
    """Every cell occupied: the span runs from the first lattice interval whose
    midpoint enters the box to the last whose midpoint is still inside
    (uniform lattice t_k = kΔt, exact slab in fp64)."""
    rng = np.random.default_rng(3)
    o, d = random_rays(400, rng)
    dt = float(np.float32(0.01))
    tn, tf = O.ray_bounds(np.ones(8**3, np.uint8), 1, 8, (0, 0, 0, 1, 1, 1), o, d, step=dt)
    checked = 0
    for r in range(len(o)):
        oo, dd = o[r].astype(np.float64), d[r].astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            a, b = (0 - oo) / dd, (1 - oo) / dd
        te = max(np.nanmax(np.minimum(a, b)), 0.0)
        tx = np.nanmin(np.maximum(a, b))
        if not tx > te:
            assert tn[r] == 0 and tf[r] == 0
            continue
        ke, kx = (te / dt) - 0.5, (tx / dt) - 0.5
        if min(abs(ke - round(ke)), abs(kx - round(kx))) < 1e-3:
            continue  # a midpoint within rounding of the box face: either side is valid
        k0 = int(np.ceil(ke))
        k1 = int(np.ceil(kx)) - 1
        if k1 < k0:
            assert tn[r] == 0
            continue
        assert tn[r] == np.float32(k0 * dt) and tf[r] == np.float32((k1 + 1) * dt)
        checked += 1
    assert checked > 200


def test_ranged_sampler_reduces_to_the_scalar_one():
    """Equal per-ray spans give exactly the scalar sampler; a culled ray yields
    uniform edges with every t at its t_near."""
    rng = np.random.default_rng(4)
    n, m = 50, 32
    e = np.sort(rng.uniform(0, 1, (n, m + 1)), axis=1)
    e[:, 0], e[:, -1] = 0.0, 1.0
    sig = rng.exponential(3.0, (n, m))
    for map_kind in (0, 1):
        ref = O.importance_sample(e, 24, sigma=sig, map_kind=map_kind, t_near=0.2, t_far=6.0)
        got = O.importance_sample_ranged(e, 24, np.full(n, 0.2), np.full(n, 6.0), sigma=sig, map_kind=map_kind)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    tn = np.full(n, 0.2)
    tf = np.full(n, 6.0)
    tn[7] = tf[7] = 0.0
    s_out, t_out = O.importance_sample_ranged(e, 24, tn, tf, sigma=sig, map_kind=1)
    assert np.allclose(s_out[7], np.linspace(0, 1, 25), rtol=0, atol=1e-15) and not t_out[7].any()


def test_ranged_identity_map_is_affine():
    """Identity map: t = t_n + s (t_f − t_n), so a span [t_n, t_f] with density σ
    has the s-space CDF of the unit span with density σ (t_f − t_n)."""
    rng = np.random.default_rng(5)
    n, m = 40, 20
    e = np.tile(np.linspace(0, 1, m + 1), (n, 1))
    sig = rng.exponential(2.0, (n, m))
    tn = rng.uniform(0.1, 2.0, n)
    tf = tn + rng.uniform(0.05, 3.0, n)
    s_a, t_a = O.importance_sample_ranged(e, 16, tn, tf, sigma=sig, map_kind=0)
    s_b, _ = O.importance_sample_ranged(e, 16, np.zeros(n), np.ones(n), sigma=sig * (tf - tn)[:, None], map_kind=0)
    assert np.allclose(s_a, s_b, rtol=0, atol=1e-12)
    assert np.allclose(t_a, tn[:, None] + s_a * (tf - tn)[:, None], rtol=1e-14, atol=1e-14)


def test_combined_shrinks_cfg1_rays():
    """CFG1 (sphere occupancy): the grid culls the rays that miss the sphere's
    cells and every kept span lies inside the unit box chord."""
    c = W.cfg1()
    tn, tf = O.ray_bounds(c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step)
    pk, _, _, _ = O.march(c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step)
    alive = tf > tn
    assert np.array_equal(alive, pk[:, 1] > 0)
    assert alive.sum() >= 20 and (~alive).sum() >= 4
    for r in np.nonzero(alive)[0]:  # each span lies within the ray's box chord (± one step)
        oo, dd = c.rays_o[r].astype(np.float64), c.rays_d[r].astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            a, b = (0 - oo) / dd, (1 - oo) / dd
        te, tx = max(np.nanmax(np.minimum(a, b)), 0.0), np.nanmin(np.maximum(a, b))
        assert te - c.step <= tn[r] < tf[r] <= tx + c.step
