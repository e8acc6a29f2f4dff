"""Pins for the proposal-supervision (PDF-matching) loss oracle (reading #21,
[ext] form): closed forms, the histogram-bound property
and finite differences -- never values the oracle produced itself."""
import numpy as np

import oracle as O


def hist(rng, n, m, lo=0.0, hi=1.0):
    e = np.sort(rng.uniform(lo, hi, (n, m + 1)), axis=1)
    e[:, 0], e[:, -1] = lo, hi
    w = rng.dirichlet(np.ones(m), n) * rng.uniform(0.2, 1.0, (n, 1))
    return e, w


def test_self_bound_is_zero():
    """The proposal equal to the final histogram bounds it exactly (B_i ≥ w_i
    with equality from the bin itself): zero loss and zero gradient."""
    rng = np.random.default_rng(1)
    t, w = hist(rng, 20, 16)
    assert np.all(O.pdf_loss(t, w, t, w) == 0)
    assert np.all(O.pdf_loss_bwd(t, w, t, w, np.ones(20)) == 0)


def test_single_proposal_bin_closed_form():
    """One proposal interval covering the ray with weight W: B_i = W for all i,
    loss = Σ max(0, w_i − W)² / (w_i + ε), g_W = −2 Σ max(0, w_i − W) / (w_i + ε)."""
    rng = np.random.default_rng(2)
    t, w = hist(rng, 10, 12)
    W = rng.uniform(0.0, 0.2, 10)
    th = np.tile([0.0, 1.0], (10, 1))
    eps = 1e-7
    res = np.maximum(0, w - W[:, None])
    assert np.allclose(O.pdf_loss(t, w, th, W[:, None], eps), (res**2 / (w + eps)).sum(1), rtol=1e-14, atol=0)
    g = O.pdf_loss_bwd(t, w, th, W[:, None], np.full(10, 0.5), eps)
    assert np.allclose(g[:, 0], 0.5 * -2 * (res / (w + eps)).sum(1), rtol=1e-14, atol=0)


def test_coarsening_bounds_the_fine_histogram():
    """Mip-NeRF 360's premise: a proposal whose bins are unions of final bins,
    each carrying the summed weight, upper-bounds every final bin -> zero loss;
    shaving weight off a proposal bin makes exactly its final bins pay."""
    rng = np.random.default_rng(3)
    t, w = hist(rng, 8, 24)
    th = t[:, ::4]  # 6 proposal bins of 4 final bins each
    wh = w.reshape(8, 6, 4).sum(2)
    assert np.all(O.pdf_loss(t, w, th, wh) == 0)
    wh2 = wh.copy()
    wh2[:, 2] = 0.0  # final bins 8..11 now only see their own proposal bin -> bound 0
    eps = 1e-7
    ref = (w[:, 8:12] ** 2 / (w[:, 8:12] + eps)).sum(1)
    assert np.allclose(O.pdf_loss(t, w, th, wh2, eps), ref, rtol=1e-12, atol=0)


def test_backward_finite_differences():
    rng = np.random.default_rng(4)
    t, w = hist(rng, 5, 20)
    th, wh = hist(rng, 5, 9)
    wh *= 0.6  # make some bins violate the bound
    g = O.pdf_loss_bwd(t, w, th, wh, np.ones(5))
    h = 1e-7
    for r in range(5):
        for j in range(9):
            a, b = wh.copy(), wh.copy()
            a[r, j] += h
            b[r, j] -= h
            fd = (O.pdf_loss(t, w, th, a)[r] - O.pdf_loss(t, w, th, b)[r]) / (2 * h)
            assert abs(g[r, j] - fd) <= 1e-5 * (1 + abs(fd)), (r, j, g[r, j], fd)
