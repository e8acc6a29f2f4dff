"""Golden worked examples (tests/golden/worked_examples.json) run through the oracle.

Each fixture carries its citation (PAPER.md / SPEC.md line); the expected values are closed
forms written into the fixture by hand, so these pin the oracle to something other than itself.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

_G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _num(v):
    return math.inf if v == "inf" else float(v)


@pytest.mark.parametrize("ex", _G["ray_aabb"], ids=lambda e: e["cite"][:6])
def test_ray_aabb(ex):
    got = O.ray_aabb(ex["o"], ex["d"], ex["lo"], ex["hi"], ex["near"], ex["far"])
    if ex["expect"] is None:
        assert got is None
    else:
        assert got is not None and np.allclose(got, ex["expect"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("ex", _G["contract"], ids=lambda e: e["cite"][:6])
def test_contract_roundtrip(ex):
    tn, tf = _num(ex["t_near"]), _num(ex["t_far"])
    t = O.contract(ex["map"], ex["s"], tn, tf)
    assert t == pytest.approx(ex["t"], rel=1e-9)
    assert O.uncontract(ex["map"], ex["t"], tn, tf) == pytest.approx(ex["s"], rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("ex", _G["render"], ids=lambda e: e["cite"][:6])
def test_render(ex):
    n = len(ex["t0"])
    pk = np.array([[0, n]], np.int64)
    out = O.render_fwd(pk, ex["t0"], ex["t1"], ex["sigma"], np.array(ex["rgb"], np.float64))
    if "weights" in ex:
        assert np.allclose(out["weights"], ex["weights"], rtol=1e-14, atol=0)
    assert np.allclose(out["color"][0], ex["color"], rtol=1e-14, atol=0)
    assert out["opacity"][0] == pytest.approx(ex["opacity"], rel=1e-14)
    if "depth" in ex:
        assert out["depth"][0] == pytest.approx(ex["depth"], rel=1e-14)
    # Eq. 2 bookkeeping the examples imply: weights sum to opacity, T_final = 1 - opacity
    assert out["weights"].sum() == pytest.approx(ex["opacity"], rel=1e-14)


@pytest.mark.parametrize("ex", _G["transmittance_cdf"], ids=lambda e: e["cite"][:6])
def test_transmittance_cdf(ex):
    T = np.array(ex["T"])
    assert np.allclose(T, ex["printed_T"], rtol=0, atol=5e-5)  # the SPEC's printed 4-digit values
    F = O.importance_cdf([ex["edges"]], sigma=[ex["sigma"]], map_kind=0, t_near=0.0, t_far=1.0)
    assert np.allclose(F[0], (1 - T) / (1 - T[-1]), rtol=0, atol=1e-15)


@pytest.mark.parametrize("ex", _G["inverse_cdf"], ids=lambda e: e["cite"][:6])
def test_inverse_cdf(ex):
    _, t = O.importance_sample([ex["edges"]], ex["n_out"], cdf=[ex["cdf"]], map_kind=ex["map"],
                               t_near=ex["t_near"], t_far=ex["t_far"])
    assert t[0].tolist() == ex["t_out"]


@pytest.mark.parametrize("ex", _G["binarize"], ids=lambda e: e["cite"][:6])
def test_binarize(ex):
    cached = np.zeros(8, np.float32)
    cached[: len(ex["cached"])] = ex["cached"]
    # decay 1 leaves the cached density unchanged, so only the threshold acts
    d, bits, _ = O.occgrid_update(1, 2, [0, 0, 0, 1, 1, 1], cached, np.zeros(8, np.float32), rule=0, decay=1.0,
                                  threshold=ex["tau"])
    assert np.array_equal(d, cached)
    assert bits[: len(ex["bits"])].tolist() == ex["bits"]


@pytest.mark.parametrize("ex", _G["ema"], ids=lambda e: e["cite"][:6])
def test_ema(ex):
    d = np.zeros(8, np.float32)
    fresh = np.full(8, ex["sigma_star"], np.float32)
    for _ in range(ex["k"]):
        d, _, _ = O.occgrid_update(1, 2, [0, 0, 0, 1, 1, 1], d, fresh, rule=0, decay=ex["gamma"], threshold=0.01)
    assert np.all(d == np.float32(ex["cached"]))


def test_early_stop_constant():
    ex = _G["early_stop"][0]
    assert -math.log(float(np.float32(ex["eps_f32"]))) == ex["neg_log_eps"]
    # the kept prefix ends at the first entering optical depth above L_eps: a ray of
    # unit-optical-depth intervals enters sample i at S_i = i, so it keeps i = 0..9 (S_9 = 9 <= 9.21 <
    # S_10): ceil(L_eps) = 10 samples
    pk = np.array([[0, 20]], np.int64)
    t0 = np.arange(20, dtype=np.float32)
    counts, _ = O.filter_counts(pk, t0, t0 + 1, np.ones(20, np.float32), ex["neg_log_eps"])
    assert counts.tolist() == [math.ceil(ex["neg_log_eps"])]


@pytest.mark.parametrize("ex", _G["accumulate"], ids=lambda e: e["cite"][:6])
def test_accumulate(ex):
    """accumulate_along_rays (Alg. 1 outputs) on the S:410-418 worked examples."""
    n = len(ex["weights"])
    pk = np.array([[0, n]], np.int64)
    w = np.array(ex["weights"], np.float64)
    v = np.array(ex["values"], np.float64).reshape(n, 3)
    out = O.accumulate(pk, w, v)
    assert np.allclose(out[0], ex["out"], rtol=1e-15, atol=0)
    op = O.accumulate(pk, w, None)
    assert op[0, 0] == pytest.approx(ex["opacity"], rel=1e-15, abs=0)


@pytest.mark.parametrize("ex", _G["accumulate_bwd"], ids=lambda e: e["cite"][:6])
def test_accumulate_bwd(ex):
    n = len(ex["weights"])
    pk = np.array([[0, n]], np.int64)
    gw, gv = O.accumulate_bwd(pk, ex["weights"], np.array(ex["values"], np.float64), np.array([ex["g_out"]], np.float64))
    assert np.allclose(gw, ex["g_weights"], rtol=1e-15, atol=0)
    assert np.allclose(gv, ex["g_values"], rtol=1e-15, atol=0)
