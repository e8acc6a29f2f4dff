"""Pins for the oracle's alpha-compositing path (P:61,
P:167): closed forms, the equivalence with the (separately pinned) density
path, telescoping, and finite differences of the forward -- never values the
oracle produced itself."""
import math

import numpy as np

import oracle as O

L_EPS = -math.log(float(np.float32(1e-4)))


def packed(counts):
    counts = np.asarray(counts, np.int64)
    start = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    return np.stack([start, counts], 1)


def random_alpha_rays(rng, n_rays=40, max_count=60):
    counts = rng.integers(0, max_count, n_rays)
    counts[0] = 0
    pk = packed(counts)
    a = rng.uniform(0.0, 0.6, counts.sum())
    return pk, a


def test_constant_alpha_closed_form():
    """α constant along a ray: T_i = (1 − α)^i, w_i = α (1 − α)^i."""
    for alpha in (0.0, 0.1, 0.5, 1.0):
        n = 9
        w, T = O.weights_alpha_fwd(packed([n]), np.full(n, alpha))
        i = np.arange(n)
        assert np.allclose(T, (1 - alpha) ** i, rtol=1e-15, atol=0)
        assert np.allclose(w, alpha * (1 - alpha) ** i, rtol=1e-15, atol=0)


def test_equals_density_path():
    """α_i = 1 − e^{−σ_i δ_i} makes alpha compositing the density path (Eq. 2):
    the product of e^{−s_j} equals e^{−Σ s_j}, so w and T agree with the
    density oracle (a different formula: exp of a sum) to rounding -- which
    here is 1 − α ≈ e^{−s} losing up to ulp/(1 − α) relative for opaque
    samples (s up to 15: ~1e-10)."""
    rng = np.random.default_rng(1)
    counts = rng.integers(0, 50, 30)
    pk = packed(counts)
    N = counts.sum()
    t0 = np.sort(rng.uniform(0, 2, N)).astype(np.float32)
    t1 = (t0 + rng.uniform(0.001, 0.05, N)).astype(np.float32)
    sig = rng.choice([0.0, 1.0, 30.0, 300.0], N).astype(np.float32) * rng.uniform(0, 1, N).astype(np.float32)
    s = sig.astype(np.float64) * (t1.astype(np.float64) - t0.astype(np.float64))
    alpha = -np.expm1(-s)
    ref = O.render_fwd(pk, t0, t1, sig, None)
    w, T = O.weights_alpha_fwd(pk, alpha)
    assert np.allclose(w, ref["weights"], rtol=1e-9, atol=1e-15)
    big = ref["trans"] > 1e-250  # below that the subnormal range loses relative precision
    assert np.allclose(T[big], ref["trans"][big], rtol=1e-9, atol=0)
    assert np.all(T[~big] < 1e-240)
    # the backward chain rule dα/dσ = δ e^{−s} links the two gradients
    gw = rng.normal(size=N)
    gT = rng.normal(size=N)
    ga = O.weights_alpha_bwd(pk, alpha, gw, gT)
    gs = O.weights_bwd(pk, t0, t1, sig, gw, gT)
    delta = t1.astype(np.float64) - t0.astype(np.float64)
    assert np.allclose(ga * delta * np.exp(-s), gs, rtol=1e-9, atol=1e-12)


def test_telescoping_sum():
    """Σ_i w_i = 1 − T_end without early stop."""
    rng = np.random.default_rng(2)
    pk, a = random_alpha_rays(rng)
    w, T = O.weights_alpha_fwd(pk, a)
    for s, c in pk:
        if c:
            t_end = T[s + c - 1] * (1 - a[s + c - 1])
            assert abs(w[s:s + c].sum() - (1 - t_end)) < 1e-14


def _loss(pk, a, gw, gT, L=np.inf):
    w, T = O.weights_alpha_fwd(pk, a, L)
    return float(np.dot(gw, w) + np.dot(gT, T))


def test_backward_finite_differences():
    """g_α against central differences of L = Σ g_w w + Σ g_T T."""
    rng = np.random.default_rng(3)
    pk, a = random_alpha_rays(rng, n_rays=6, max_count=25)
    a = np.clip(a, 0.05, 0.9)
    gw = rng.normal(size=len(a))
    gT = rng.normal(size=len(a))
    ga = O.weights_alpha_bwd(pk, a, gw, gT)
    h = 1e-6
    for k in range(len(a)):
        ap, am = a.copy(), a.copy()
        ap[k] += h
        am[k] -= h
        fd = (_loss(pk, ap, gw, gT) - _loss(pk, am, gw, gT)) / (2 * h)
        assert abs(ga[k] - fd) <= 1e-6 * (1 + abs(fd)), (k, ga[k], fd)


def test_opaque_sample_is_zero_safe():
    """α_k = 1: everything behind is hidden (T = w = 0) and the gradient stays
    finite and equal to the finite difference of the forward.  L is affine in
    each α_k, so a one-sided difference inside [0, 1] is exact up to rounding
    (α_k > 1 would make T negative, outside the method's domain)."""
    a = np.array([0.3, 0.2, 1.0, 0.4, 0.7])
    pk = packed([5])
    w, T = O.weights_alpha_fwd(pk, a)
    assert T[3] == 0 and T[4] == 0 and w[3] == 0 and w[4] == 0
    gw = np.array([0.5, -1.0, 2.0, 3.0, -4.0])
    ga = O.weights_alpha_bwd(pk, a, gw)
    assert np.all(np.isfinite(ga))
    h = 1e-6
    for k in range(5):
        am = a.copy()
        am[k] -= h
        fd = (_loss(pk, a, gw, np.zeros(5)) - _loss(pk, am, gw, np.zeros(5))) / h
        assert abs(ga[k] - fd) <= 1e-6 * (1 + abs(fd))
    # samples behind the opaque one receive gradient only through w, which is 0 there
    assert ga[3] == 0 and ga[4] == 0


def test_early_stop():
    """w_i = 0 from the first T_i < ε_T on; the mask is a constant for the backward."""
    a = np.full(40, 0.3)
    pk = packed([40])
    eps_T = math.exp(-L_EPS)
    w, T = O.weights_alpha_fwd(pk, a, L_EPS)
    first_dead = int(np.argmax(0.7 ** np.arange(40) < eps_T))
    assert first_dead > 0
    assert np.all(w[first_dead:] == 0) and np.all(w[:first_dead] > 0)
    gw = np.linspace(-1, 1, 40)
    ga = O.weights_alpha_bwd(pk, a, gw, None, L_EPS)
    h = 1e-7  # small enough that no liveness decision flips (margins are ~1e-2 relative)
    for k in (0, 5, first_dead - 1, first_dead, 39):
        ap, am = a.copy(), a.copy()
        ap[k] += h
        am[k] -= h
        fd = (_loss(pk, ap, gw, np.zeros(40), L_EPS) - _loss(pk, am, gw, np.zeros(40), L_EPS)) / (2 * h)
        assert abs(ga[k] - fd) <= 1e-6 * (1 + abs(fd))
