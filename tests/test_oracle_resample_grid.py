"""Pins for the oracle's inverse-CDF resampler (O8) and occupancy-grid update (O9)."""
import math

import numpy as np
import pytest

import oracle as O


# ----------------------------------------------------------------------------- resample (Eq. 1, Eq. 3)
def test_uniform_profile_spec_example():
    """uniform profile on t in [2,6], u = 0.5 -> t = 4 (identity Φ)."""
    s, t = O.importance_sample([[0.0, 1.0]], 2, cdf=[[0.0, 1.0]], map_kind=0, t_near=2.0, t_far=6.0)
    assert s[0].tolist() == [0.0, 0.5, 1.0]
    assert t[0].tolist() == [2.0, 4.0, 6.0]


def test_constant_sigma_cdf_closed_form():
    """constant σ = 1 over t in [0,1], 4 bins: T = {1, e^-.25, e^-.5, e^-.75, e^-1};
    the sampler's CDF is F = 1 - T (Eq. 3), normalised by F(t_f)."""
    F = O.importance_cdf([[0, 0.25, 0.5, 0.75, 1.0]], sigma=[[1.0] * 4], map_kind=0, t_near=0.0, t_far=1.0)
    T = np.array([1, 0.7788007830714049, 0.6065306597126334, 0.4723665527410147, 0.36787944117144233])
    assert np.allclose(F[0], (1 - T) / (1 - T[-1]), rtol=0, atol=1e-15)
    assert abs(T[1] - 0.7788) < 1e-4 and abs(T[4] - 0.3679) < 1e-4


def _interp_cdf(s, e, F):
    return np.interp(s, e, F)


def _cdf_from_definition(e, sig, map_kind, tn, tf):
    """F = 1 - T with T = exp(-Σ σ δ) (Eq. 2/3), normalised; piecewise linear in s."""
    t = np.array([O.contract(map_kind, float(x), tn, tf) for x in e])
    S = np.concatenate([[0.0], np.cumsum(np.asarray(sig, np.float64) * np.diff(t))])
    F = -np.expm1(-S)
    return F / F[-1]


@pytest.mark.parametrize("map_kind", [0, 1])
def test_backward_error_and_monotone(map_kind):
    """Each output edge inverts the CDF: F̂(s_i) = u_i; edges non-decreasing;
    first/last edges at the ends of the mass."""
    rng = np.random.default_rng(0)
    n_rays, m, n = 40, 64, 24
    e = np.sort(rng.uniform(0, 1, (n_rays, m + 1)), axis=1)
    e[:, 0], e[:, -1] = 0.0, 1.0
    sig = np.where(rng.random((n_rays, m)) < 0.5, 0.0, rng.uniform(0, 30, (n_rays, m)))
    sig[:, :3] = 0.0
    sig[:, -2:] = 0.0
    tn, tf = (0.2, 1000.0) if map_kind else (2.0, 6.0)
    s_out, t_out = O.importance_sample(e, n, sigma=sig, map_kind=map_kind, t_near=tn, t_far=tf)
    for r in range(n_rays):
        F = _cdf_from_definition(e[r], sig[r], map_kind, tn, tf)
        u = np.arange(n + 1) / n
        assert np.abs(_interp_cdf(s_out[r], e[r], F) - u).max() < 1e-9
        assert np.all(np.diff(s_out[r]) >= 0)
        first = np.nonzero(sig[r] > 0)[0]
        assert s_out[r, 0] == e[r, first[0]]  # u = 0: start of the mass
        assert s_out[r, -1] == e[r, np.argmax(F >= 1.0)]  # u = 1: where F̂ first reaches 1
        assert s_out[r, -1] <= e[r, first[-1] + 1]
        for k in range(n + 1):
            assert abs(t_out[r, k] - O.contract(map_kind, s_out[r, k], tn, tf)) <= 1e-12 * t_out[r, k]


def test_stratified_one_sample_per_stratum_and_ks():
    """stratified draws on a uniform profile land exactly one per stratum;
    S:368: the empirical CDF of draws matches F̂ (KS < 0.01)."""
    n = 999
    s, _ = O.importance_sample([[0.0, 1.0]], n, cdf=[[0.0, 1.0]], map_kind=0, t_near=0, t_far=1,
                               stratified=1, seed=11)
    k = np.floor(s[0] * (n + 1)).astype(int)
    assert np.array_equal(k, np.arange(n + 1))
    rng = np.random.default_rng(1)
    m = 32
    e = np.linspace(0, 1, m + 1)[None]
    sig = rng.uniform(0, 5, (1, m))
    s, _ = O.importance_sample(e, 100000 - 1, sigma=sig, map_kind=0, t_near=0, t_far=1, stratified=1, seed=3)
    F = _cdf_from_definition(e[0], sig[0], 0, 0.0, 1.0)
    emp = (np.arange(1, s.shape[1] + 1)) / s.shape[1]
    ks = np.abs(emp - np.interp(np.sort(s[0]), e[0], F)).max()
    assert ks < 0.01


def test_zero_mass_gives_uniform_edges():
    """reading #16: F(t_f) <= 1e-12 -> uniform edges in s."""
    e = np.linspace(0.1, 0.9, 9)[None]
    s, _ = O.importance_sample(e, 4, sigma=np.zeros((1, 8)), map_kind=1)
    assert np.allclose(s[0], np.linspace(0.1, 0.9, 5), rtol=0, atol=1e-15)


def test_single_massive_bin():
    """all mass in one bin: every output edge lies in that bin, evenly spaced in s."""
    e = np.linspace(0, 1, 9)[None]
    sig = np.zeros((1, 8))
    sig[0, 3] = 7.0
    s, _ = O.importance_sample(e, 8, sigma=sig, map_kind=0, t_near=0, t_far=1)
    assert np.allclose(s[0], np.linspace(3 / 8, 4 / 8, 9), rtol=0, atol=1e-15)


# ----------------------------------------------------------------------------- grid update
ROI = (0, 0, 0, 1, 1, 1)


def test_ema_geometric_series():
    """S:257 / S:284: static field, zero jitter, from 0: occ_k = σ*(1 - γ^k)
    (fp32 state: within k·2^-24 relative)."""
    rng = np.random.default_rng(0)
    fresh = rng.uniform(0, 10, 4**3).astype(np.float32)
    for gam in (0.5, 0.95):
        dens = np.zeros(4**3, np.float32)
        for k in range(1, 51):
            dens, bits, _ = O.occgrid_update(1, 4, ROI, dens, fresh, decay=gam, threshold=0.01)
            expect = fresh.astype(np.float64) * (1 - gam**k)
            assert np.all(np.abs(dens - expect) <= k * 2.0**-23 * fresh + 1e-30)
            assert np.all(np.abs(dens - fresh) <= fresh * gam**k * (1 + 1e-6) + k * 2.0**-23 * fresh)


def test_update_degenerate_cases():
    fresh = np.array([0, 1, 2, 3, 0.5, 0, 7, 8], np.float32)
    d0 = np.array([5, 5, 5, 5, 5, 5, 5, 5], np.float32)
    d, b, _ = O.occgrid_update(1, 2, ROI, d0, fresh, decay=0.0)  # S:258 γ = 0 -> instantaneous query
    assert np.array_equal(d, fresh)
    d, b, _ = O.occgrid_update(1, 2, ROI, np.zeros(8, np.float32), np.zeros(8, np.float32))
    assert not d.any() and not b.any()
    tau = np.float32(0.25)
    d, b, _ = O.occgrid_update(1, 2, ROI, np.zeros(8, np.float32),
                               np.array([0, tau, 2 * tau, 0, tau, 2 * tau, 0, 0], np.float32),
                               decay=0.0, threshold=float(tau))  # S:266 strict >
    assert b.tolist() == [0, 0, 1, 0, 0, 1, 0, 0]
    d2, b2, _ = O.occgrid_update(1, 2, ROI, d, np.zeros(8, np.float32), decay=1.0, threshold=float(tau))
    assert np.array_equal(d2, d) and np.array_equal(b2, b)  # S:268 binarize idempotent
    d, b, _ = O.occgrid_update(1, 2, ROI, np.zeros(8, np.float32), fresh, rule=1, decay=0.95)
    assert np.array_equal(d, fresh)  # max-decay with a static field: σ* after one update


def test_min_mean_threshold():
    fresh = np.array([0, 0, 0, 0, 0, 0, 0, 0.08], np.float32)
    d, b, mean = O.occgrid_update(1, 2, ROI, np.zeros(8, np.float32), fresh, decay=0.0, threshold=0.5,
                                  thresh_rule=1)
    assert abs(mean - 0.01) < 1e-9 and b.tolist() == [0] * 7 + [1]


def test_points_cell_centres_and_jitter():
    levels, R = 2, 4
    roi = (-1, -1, -1, 1, 1, 1)
    xyz = O.occgrid_points(levels, R, roi, seed=1, step=0, jitter=0)
    i = np.arange(R**3)
    ijk = np.stack([i % R, (i // R) % R, i // R**2], 1)
    assert np.array_equal(xyz[: R**3], (-1 + (ijk + 0.5) * 0.5).astype(np.float32))
    assert np.array_equal(xyz[R**3 :], (-2 + (ijk + 0.5) * 1.0).astype(np.float32))
    xj = O.occgrid_points(levels, R, roi, seed=1, step=3, jitter=1)
    lo = np.concatenate([-1 + ijk * 0.5, -2 + ijk * 1.0])
    w = np.concatenate([np.full((R**3, 3), 0.5), np.full((R**3, 3), 1.0)])
    assert np.all(xj >= lo) and np.all(xj <= lo + w)
    assert not np.array_equal(xj, O.occgrid_points(levels, R, roi, seed=1, step=4, jitter=1))
    # sub-range = slice of the full range
    part = O.occgrid_points(levels, R, roi, seed=1, step=3, jitter=1, cell_begin=70, cell_count=20)
    assert np.array_equal(part, xj[70:90])


def test_constant_box_eighth_occupancy():
    """a ConstantBox covering 1/8 of the volume gives occupied fraction 0.125."""
    R = 16
    xyz = O.occgrid_points(1, R, ROI, seed=0, step=0, jitter=0)
    fresh = np.where(np.all(xyz < 0.5, axis=1), 3.0, 0.0).astype(np.float32)
    d, b, _ = O.occgrid_update(1, R, ROI, np.zeros(R**3, np.float32), fresh, decay=0.0, threshold=1.0)
    assert b.mean() == 0.125


def test_owner_computes_max_merge_equals_single_rank():
    """reading #25: ranks evaluate disjoint owner slabs; non-owners contribute 0;
    the element-wise MAX of the rank buffers equals the one-rank fresh buffer,
    so the update is bit-identical for any rank count."""
    rng = np.random.default_rng(3)
    n = 3 * 8**3
    fresh = rng.uniform(0, 2, n).astype(np.float32)
    dens = rng.uniform(0, 2, n).astype(np.float32)
    ref = O.occgrid_update(3, 8, ROI, dens, fresh, decay=0.95, threshold=0.5)
    for G in (2, 3, 8):
        bufs = []
        for g in range(G):
            b = np.zeros(n, np.float32)
            lo, hi = g * n // G, (g + 1) * n // G
            b[lo:hi] = fresh[lo:hi]
            bufs.append(b)
        merged = np.maximum.reduce(bufs)
        got = O.occgrid_update(3, 8, ROI, dens, merged, decay=0.95, threshold=0.5)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def test_dynamic_timestamps_uniform_and_reproducible():
    """reading #20: per-cell timestamps on the 2^-24 grid in [0, 1), uniform
    (KS), independent across draws, sub-ranges are slices of the full range."""
    from scipy import stats

    R = 32
    t0 = O.occgrid_times(1, R, ROI, seed=7, step=16, draw=0)
    t1 = O.occgrid_times(1, R, ROI, seed=7, step=16, draw=1)
    for t in (t0, t1):
        assert t.min() >= 0 and t.max() < 1
        assert np.array_equal(t * 2.0**24, np.floor(t * 2.0**24))
        assert stats.kstest(t.astype(np.float64), "uniform").pvalue > 1e-3
    assert abs(np.corrcoef(t0, t1)[0, 1]) < 0.03
    assert np.array_equal(O.occgrid_times(1, R, ROI, seed=7, step=16, draw=1, cell_begin=100, cell_count=50),
                          t1[100:150])
    assert not np.array_equal(t0, O.occgrid_times(1, R, ROI, seed=7, step=32, draw=0))


def test_dynamic_grid_holds_the_max_over_time():
    """the shared grid marks the maximum opacity over all timestamps.  A
    sphere moving along x over t in [0, 1): cells it covers at every t are
    occupied after one draw, cells it never reaches never are, and with many
    draws the occupied set approaches the swept volume."""
    R = 32
    xyz = O.occgrid_points(1, R, ROI, seed=0, step=0, jitter=0).astype(np.float64)

    rad = 0.25

    def sigma(x, t):  # radius 0.25, centre (0.35 + 0.3 t, 0.5, 0.5)
        c = np.stack([0.35 + 0.3 * t, np.full_like(t, 0.5), np.full_like(t, 0.5)], 1)
        return np.where(np.linalg.norm(x - c, axis=1) < rad, 10.0, 0.0).astype(np.float32)

    fresh = None
    for j in range(48):
        v = sigma(xyz, O.occgrid_times(1, R, ROI, seed=3, step=0, draw=j).astype(np.float64))
        fresh = v if fresh is None else np.maximum(fresh, v)
    _, bits, _ = O.occgrid_update(1, R, ROI, np.zeros(R**3, np.float32), fresh, decay=0.0, threshold=1.0)
    dy = np.linalg.norm(xyz[:, 1:] - 0.5, axis=1)
    # |x − c(t)|² is convex in t, so a point inside at t = 0 and at t = 1 is inside for every t
    c0, c1 = np.array([0.35, 0.5, 0.5]), np.array([0.65, 0.5, 0.5])
    always = (np.linalg.norm(xyz - c0, axis=1) < rad - 1e-3) & (np.linalg.norm(xyz - c1, axis=1) < rad - 1e-3)
    never = np.linalg.norm(np.stack([np.clip(xyz[:, 0], 0.35, 0.65) - xyz[:, 0], dy], 1), axis=1) > rad
    assert always.sum() > 0 and np.all(bits[always] == 1)
    assert np.all(bits[never] == 0)
    swept = ~never
    assert bits[swept].mean() > 0.9  # 48 draws cover nearly the whole swept volume
