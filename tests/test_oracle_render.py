"""Pins for the oracle's filter, transmittance/weights, accumulation and
backward (O5-O7, O10).  Values come from SPEC worked examples, closed forms,
finite differences and invariants -- never from the oracle itself."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

L_EPS = -math.log(float(np.float32(1e-4)))


def packed(counts):
    counts = np.asarray(counts, np.int64)
    start = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    return np.stack([start, counts], 1)


def chain(widths, t_start=0.0):
    e = t_start + np.concatenate([[0.0], np.cumsum(widths)])
    return e[:-1], e[1:]


# ----------------------------------------------------------------------------- render fwd
def test_single_interval_spec_example():
    """one interval, σ·δ = 1, c = (1,1,1) -> α = 1 - e^-1 ≈ 0.63212."""
    out = O.render_fwd(packed([1]), [0.0], [1.0], [1.0], [[1, 1, 1]])
    a = 1 - math.exp(-1)
    assert abs(out["opacity"][0] - a) < 1e-15 and np.allclose(out["color"][0], a, atol=1e-15, rtol=0)
    assert abs(a - 0.63212) < 1e-5
    assert out["depth"][0] == 0.5


def test_zero_density_spec_example():
    """σ ≡ 0 -> color 0, opacity 0, depth 0."""
    t0, t1 = chain([0.1] * 7)
    out = O.render_fwd(packed([7]), t0, t1, np.zeros(7), np.ones((7, 3)))
    assert out["opacity"][0] == 0 and out["depth"][0] == 0 and not out["color"].any()


def test_two_half_alphas_spec_example():
    """α1 = α2 = 0.5 -> weights {0.5, 0.25}, opacity 0.75."""
    out = O.render_fwd(packed([2]), [0.0, 1.0], [1.0, 2.0], [math.log(2)] * 2, np.ones((2, 3)))
    assert np.allclose(out["weights"], [0.5, 0.25], atol=1e-15, rtol=0)
    assert abs(out["opacity"][0] - 0.75) < 1e-15


def test_constant_density_chord_closed_form():
    """Eq. 2/3: T_final = exp(-σL); opacity = 1 - T_final = Σ w."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 400))
        w = rng.uniform(1e-3, 2e-2, n)
        t0, t1 = chain(w, rng.uniform(0, 1))
        sig = float(rng.uniform(0.1, 50))
        out = O.render_fwd(packed([n]), t0, t1, np.full(n, sig), rng.uniform(0, 1, (n, 3)))
        L = float(np.sum(np.asarray(t1) - np.asarray(t0)))
        assert abs(out["opacity"][0] - (1 - math.exp(-sig * L))) < 1e-13
        assert abs(out["weights"].sum() - out["opacity"][0]) < 1e-13
        assert abs(out["trans"][0] - 1.0) == 0.0


def test_splitting_invariance():
    """splitting intervals of a constant-σ field leaves color/opacity unchanged (1e-12)."""
    rng = np.random.default_rng(1)
    for _ in range(10):
        n = int(rng.integers(1, 50))
        t0, t1 = chain(rng.uniform(0.01, 0.1, n))
        sig = rng.uniform(0, 20, n)
        col = rng.uniform(0, 1, (n, 3))
        a = O.render_fwd(packed([n]), t0, t1, sig, col)
        mid = (t0 + t1) / 2
        t0s = np.stack([t0, mid], 1).ravel()
        t1s = np.stack([mid, t1], 1).ravel()
        b = O.render_fwd(packed([2 * n]), t0s, t1s, np.repeat(sig, 2), np.repeat(col, 2, 0))
        assert abs(a["opacity"][0] - b["opacity"][0]) < 1e-12
        assert np.abs(a["color"] - b["color"]).max() < 1e-12


def test_quadrature_limit():
    """n_quad -> inf gives opacity -> 1 - e^{-σ0 ℓ} (within 1e-4 at 2^14, σ0ℓ <= 5),
    and the quadrature error shrinks monotonically."""
    box = [-0.5, -0.5, -0.5, 0.5, 0.5, 0.5]
    for s0 in (1.0, 3.0, 5.0):
        o, d = (-1.0, 0.1, 0.2), (1.0, 0.0, 0.0)  # chord length 1
        op, dp = O.render_quadrature(0, box, s0, o, d, 0.0, 3.0, 1 << 14)
        assert abs(op - (1 - math.exp(-s0))) < 1e-4
        errs = [abs(O.render_quadrature(0, box, s0, o, d, 0.0, 3.0, n)[0] - (1 - math.exp(-s0))) for n in (37, 74, 148, 296)]
        assert all(a >= b for a, b in zip(errs, errs[1:]))
    op, _ = O.render_quadrature(1, [0, 0, 0, 0.5], 2.0, (-2, 0, 0), (1, 0, 0), 0, 4, 1 << 14)
    assert abs(op - (1 - math.exp(-2.0))) < 1e-3


def test_render_invariants_on_fuzz():
    """0 <= w, Σw <= 1, color <= opacity; T monotone, T_0 = 1."""
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(300, seed=2)
    out = O.render_fwd(pk, t0, t1, sig, rgb)
    assert np.all(out["weights"] >= 0)
    assert np.all(out["opacity"] <= 1 + 1e-12)
    assert np.all(out["color"] <= out["opacity"][:, None] + 1e-12)
    for s, c in pk:
        if c:
            T = out["trans"][s : s + c]
            assert T[0] == 1.0 and np.all(np.diff(T) <= 0)
    # order invariance of packing: rendering rays separately matches
    for r in range(0, 300, 37):
        s, c = pk[r]
        one = O.render_fwd(packed([c]), t0[s : s + c], t1[s : s + c], sig[s : s + c], rgb[s : s + c])
        assert one["opacity"][0] == out["opacity"][r] and np.array_equal(one["color"][0], out["color"][r])


def test_depth_is_expected_midpoint():
    """reading #12: depth = Σ w·m / O; a single opaque interval gives its midpoint."""
    out = O.render_fwd(packed([3]), [1.0, 2.0, 3.0], [1.5, 2.5, 3.5], [0.0, 1e4, 0.0], np.ones((3, 3)))
    assert abs(out["depth"][0] - 2.25) < 1e-12


# ----------------------------------------------------------------------------- filter
def test_filter_spec_examples():
    # S:364 first interval σδ = 20 -> every later interval dropped
    t0, t1 = chain([0.1] * 6)
    cnt, _ = O.filter_counts(packed([6]), t0, t1, [200.0, 1, 1, 1, 1, 1], L_EPS)
    assert cnt.tolist() == [1]
    # S:363 σ ≡ 0 -> nothing dropped; S:365 threshold 0 (-ln 0 = +inf) -> identity
    cnt, _ = O.filter_counts(packed([6]), t0, t1, np.zeros(6), L_EPS)
    assert cnt.tolist() == [6]
    cnt, _ = O.filter_counts(packed([6]), t0, t1, [500.0] * 6, math.inf)
    assert cnt.tolist() == [6]


def test_filter_entering_transmittance_is_strict():
    """reading #9: drop sample i iff its ENTERING T_i < ε (S_i > -ln ε); T = ε is kept."""
    L = float(np.float32(L_EPS))
    cnt, _ = O.filter_counts(packed([3]), [0.0, 1.0, 2.0], [1.0, 2.0, 3.0], [L, 1.0, 1.0], L)
    assert cnt.tolist() == [2]


def test_filter_monotone_and_bounded_influence():
    """S:372 survivors(ε1) ⊇ survivors(ε2) for ε1 < ε2; P:86 'almost no
    influence': dropped mass <= T_cut < ε, so opacity changes by < ε."""
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(400, seed=3)
    prev = None
    for eps in (1e-8, 1e-6, 1e-4, 1e-2, 0.5):
        cnt, _ = O.filter_counts(pk, t0, t1, sig, -math.log(eps))
        if prev is not None:
            assert np.all(cnt <= prev)
        prev = cnt
        pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, -math.log(eps))
        idx = np.concatenate([np.arange(s, s + c) for (s, _), c in zip(pk, cnt) if c] or [np.zeros(0, int)])
        full = O.render_fwd(pk, t0, t1, sig, rgb)
        filt = O.render_fwd(pk2, a0, a1, sig[idx], rgb[idx])
        assert np.all(np.abs(full["opacity"] - filt["opacity"]) < eps)
        assert np.all(np.abs(full["color"] - filt["color"]) < eps)
        assert np.array_equal(a0, t0[idx]) and np.array_equal(r2, rid[idx])


def test_render_early_stop_equals_filtered_render():
    """Early stop inside render (ε) gives the same color as rendering the
    filtered packed samples (the cut is the same prefix)."""
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(200, seed=4)
    pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, L_EPS)
    cnt = pk2[:, 1]
    idx = np.concatenate([np.arange(s, s + c) for (s, _), c in zip(pk, cnt) if c])
    es = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=L_EPS)
    filt = O.render_fwd(pk2, a0, a1, sig[idx], rgb[idx])
    assert np.abs(es["color"] - filt["color"]).max() < 1e-13
    assert np.abs(es["opacity"] - filt["opacity"]).max() < 1e-13


# ----------------------------------------------------------------------------- backward
def _loss(pk, t0, t1, sig, rgb, gC, gO, gD, eps):
    out = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=eps)
    return float(np.sum(out["color"] * gC) + np.sum(out["opacity"] * gO) + np.sum(out["depth"] * gD))


@pytest.mark.parametrize("eps", [math.inf, 3.0])
def test_render_bwd_finite_differences(eps):
    """Central differences in fp64 (h = 1e-6) agree with O7 (SURVEY c.3 measured 1.2e-9)."""
    rng = np.random.default_rng(5)
    counts = [9, 0, 1, 15]
    pk = packed(counts)
    N = sum(counts)
    t0 = np.zeros(N)
    t1 = np.zeros(N)
    for (s, c) in pk:
        a, b = chain(rng.uniform(0.01, 0.2, c), rng.uniform(0, 1))
        t0[s : s + c], t1[s : s + c] = a, b
    sig = rng.uniform(0, 8, N)
    rgb = rng.uniform(0, 1, (N, 3))
    gC, gO, gD = rng.normal(size=(4, 3)), rng.normal(size=4), rng.normal(size=4)
    gs, grgb = O.render_bwd(pk, t0, t1, sig, rgb, gC, gO, gD, neg_log_eps=eps)
    h = 1e-6
    for q in range(N):
        sp, sm = sig.copy(), sig.copy()
        sp[q] += h
        sm[q] -= h
        fd = (_loss(pk, t0, t1, sp, rgb, gC, gO, gD, eps) - _loss(pk, t0, t1, sm, rgb, gC, gO, gD, eps)) / (2 * h)
        assert abs(fd - gs[q]) <= 1e-6 * max(1.0, abs(fd)), (q, fd, gs[q])
        for ch in range(3):
            rp, rm = rgb.copy(), rgb.copy()
            rp[q, ch] += h
            rm[q, ch] -= h
            fd = (_loss(pk, t0, t1, sig, rp, gC, gO, gD, eps) - _loss(pk, t0, t1, sig, rm, gC, gO, gD, eps)) / (2 * h)
            assert abs(fd - grgb[q, ch]) <= 1e-6 * max(1.0, abs(fd))


def test_single_interval_opacity_gradient_closed_form():
    """∂O/∂σ = δ·e^{-σδ} for one interval."""
    for sig, dl in ((0.5, 0.3), (10.0, 0.01), (0.0, 2.0)):
        gs, _ = O.render_bwd(packed([1]), [1.0], [1.0 + dl], [sig], [[0.2, 0.3, 0.4]], None, [1.0], None)
        assert abs(gs[0] - dl * math.exp(-sig * dl)) < 1e-14


def test_weights_bwd_finite_differences():
    rng = np.random.default_rng(6)
    n = 12
    t0, t1 = chain(rng.uniform(0.01, 0.2, n))
    sig = rng.uniform(0, 10, n)
    gw, gT = rng.normal(size=n), rng.normal(size=n)
    pk = packed([n])
    for eps in (math.inf, 2.0):
        gs = O.weights_bwd(pk, t0, t1, sig, gw, gT, neg_log_eps=eps)

        def f(s):
            out = O.render_fwd(pk, t0, t1, s, None, neg_log_eps=eps)
            return float(np.dot(out["weights"], gw) + np.dot(out["trans"], gT))

        h = 1e-6
        for q in range(n):
            sp, sm = sig.copy(), sig.copy()
            sp[q] += h
            sm[q] -= h
            fd = (f(sp) - f(sm)) / (2 * h)
            assert abs(fd - gs[q]) <= 1e-6 * max(1.0, abs(fd))


def test_accumulate_closed_forms_and_bwd():
    rng = np.random.default_rng(7)
    pk = packed([3, 0, 5])
    w = rng.uniform(0, 0.3, 8)
    v = rng.uniform(0, 1, (8, 3))
    out = O.accumulate(pk, w, v)
    assert np.allclose(out[0], (w[:3, None] * v[:3]).sum(0), rtol=0, atol=1e-15)
    assert not out[1].any()
    op = O.accumulate(pk, w, None)
    assert np.allclose(op[:, 0], [w[:3].sum(), 0, w[3:].sum()], rtol=0, atol=1e-15)
    g = rng.normal(size=(3, 3))
    gw, gv = O.accumulate_bwd(pk, w, v, g)
    assert np.allclose(gw[:3], v[:3] @ g[0], rtol=0, atol=1e-14)
    assert np.allclose(gv[3:], w[3:, None] * g[2], rtol=0, atol=1e-15)


def test_oracle_render_deterministic_across_threads():
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(500, seed=8)
    O.set_num_threads(1)
    a = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=L_EPS)
    ga = O.render_bwd(pk, t0, t1, sig, rgb, np.ones((500, 3)), np.ones(500), np.ones(500), neg_log_eps=L_EPS)
    O.set_num_threads(8)
    b = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=L_EPS)
    gb = O.render_bwd(pk, t0, t1, sig, rgb, np.ones((500, 3)), np.ones(500), np.ones(500), neg_log_eps=L_EPS)
    for k in a:
        assert np.array_equal(a[k], b[k])
    assert np.array_equal(ga[0], gb[0]) and np.array_equal(ga[1], gb[1])


def test_accumulate_equals_render_fwd_outputs():
    """Pin or_accumulate to the independently pinned O6 renderer (Eq. 2 closed forms, S:416-418
    goldens): accumulating O6's own weights with rgb, ones and interval midpoints must give O6's
    colour, opacity and depth·opacity on ragged fuzz inputs."""
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(400, seed=21)
    for eps in (math.inf, L_EPS):
        ref = O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=eps)
        w = ref["weights"]
        col = O.accumulate(pk, w, rgb)
        assert np.allclose(col, ref["color"], rtol=1e-12, atol=1e-15)
        op = O.accumulate(pk, w, None)[:, 0]
        assert np.allclose(op, ref["opacity"], rtol=1e-12, atol=1e-15)
        mid = (t0.astype(np.float64) + t1.astype(np.float64)) / 2.0
        nd = O.accumulate(pk, w, mid[:, None])[:, 0]
        assert np.allclose(nd, ref["depth"] * np.maximum(ref["opacity"], 1e-10), rtol=1e-10, atol=1e-15)


def test_accumulate_bwd_finite_differences():
    """or_accumulate_bwd against central finite differences of or_accumulate (a linear map, so the
    difference quotient is exact up to rounding)."""
    pk, t0, t1, rid, sig, rgb = W.ragged_samples(60, seed=22)
    rng = np.random.default_rng(23)
    n = len(t0)
    w = rng.uniform(0, 0.2, n)
    g = rng.normal(size=(60, 3))
    gw, gv = O.accumulate_bwd(pk, w, rgb, g)

    def f(wv, vv):
        return float((O.accumulate(pk, wv, vv) * g).sum())

    h = 1e-3
    for q in rng.choice(n, 40, replace=False):
        wp, wm = w.copy(), w.copy()
        wp[q] += h
        wm[q] -= h
        fd = (f(wp, rgb) - f(wm, rgb)) / (2 * h)
        assert abs(fd - gw[q]) <= 1e-9 * max(1.0, abs(fd))
        ch = int(rng.integers(3))
        vp, vm = rgb.astype(np.float64).copy(), rgb.astype(np.float64).copy()
        vp[q, ch] += h
        vm[q, ch] -= h
        fd = (f(w, vp) - f(w, vm)) / (2 * h)
        assert abs(fd - gv[q, ch]) <= 1e-9 * max(1.0, abs(fd))
    # ones (opacity): g_w is the ray's upstream gradient
    gw1, _ = O.accumulate_bwd(pk, w, None, g[:, :1])
    ray = np.repeat(np.arange(60), pk[:, 1])
    assert np.array_equal(gw1, g[ray, 0])
