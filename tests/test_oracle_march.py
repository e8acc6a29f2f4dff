"""Pins for the oracle's geometry and occupancy-grid marching (O1-O4).

Each test checks the oracle against something other than itself: values the
SPEC/paper print, closed forms, brute force on tiny inputs, or geometric
properties evaluated independently in fp64 numpy.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads as W

LO1 = (-1.0, -1.0, -1.0)
HI1 = (1.0, 1.0, 1.0)


# ----------------------------------------------------------------------------- RNG
def test_philox_known_answers():
    """Random123 known-answer vectors for Philox4x32-10."""
    assert O.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


# ----------------------------------------------------------------------------- O1 slab
def test_slab_spec_examples():
    assert O.ray_aabb((-2, 0, 0), (1, 0, 0), LO1, HI1, 0, 10) == (1.0, 3.0)
    assert O.ray_aabb((0, 0, 0), (1, 0, 0), LO1, HI1, 0, 10) == (0.0, 1.0)  # S:66 origin inside
    assert O.ray_aabb((-2, 5, 0), (1, 0, 0), LO1, HI1, 0, 10) is None  # S:67 miss


def test_slab_brute_force():
    """the point-inside-box predicate changes at the reported t within one step."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        o = rng.uniform(-3, 3, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        ts = np.linspace(0, 10, 10001)
        pts = o + ts[:, None] * d
        inside = np.all((pts >= -1) & (pts < 1), axis=1)
        res = O.ray_aabb(o, d, LO1, HI1, 0.0, 10.0)
        if res is None:
            assert inside.sum() <= 1
        else:
            te, tx = res
            idx = np.nonzero(inside)[0]
            assert abs(ts[idx[0]] - te) <= 1e-3 + 1e-9 and abs(ts[idx[-1]] - tx) <= 1e-3 + 1e-9


# ----------------------------------------------------------------------------- Φ
def test_contraction_spec_examples():
    assert O.contract(0, 0.5, 2.0, 6.0) == 4.0
    assert O.contract(1, 0.5, 1.0, math.inf) == 2.0
    assert abs(O.uncontract(1, 1e6, 1.0, math.inf) - 0.999999) < 1e-9
    rng = np.random.default_rng(1)
    prev = -1.0
    for s in np.sort(rng.uniform(0, 1, 1000)):
        for m, tf in ((0, 6.0), (1, 1000.0), (1, math.inf)):
            t = O.contract(m, s, 0.2 if m else 2.0, tf)
            assert abs(O.uncontract(m, t, 0.2 if m else 2.0, tf) - s) < 1e-9
        t = O.contract(1, s, 0.2, 1000.0)
        assert t > prev
        prev = t


# ----------------------------------------------------------------------------- helpers
def random_rays(n, rng, box_lo=0.0, box_hi=1.0, special=True):
    """random rays toward a box, including axis-aligned, inside-box and grazing ones"""
    c = (box_lo + box_hi) / 2
    w = box_hi - box_lo
    o = c + rng.normal(size=(n, 3)) * w * 1.5
    tgt = c + rng.uniform(-0.6, 0.6, (n, 3)) * w
    d = tgt - o
    if special and n >= 12:
        o[0], d[0] = [box_lo - 0.5 * w, c + 0.1 * w, c], [1, 0, 0]  # axis aligned
        o[1], d[1] = [c, c, c], [0.3, -0.5, 0.8]  # inside the box
        o[2], d[2] = [box_lo - 0.5 * w, box_lo, c], [1, 0, 0]  # grazing a face (on the half-open lo side)
        o[3], d[3] = [box_lo - 0.5 * w, box_hi, c], [1, 0, 0]  # grazing the hi face (excluded)
        o[4], d[4] = [c, c, box_hi + w], [0, 0, -1]  # axis aligned, -z
        o[5], d[5] = [box_lo - w, box_lo - w, box_lo - w], [1, 1, 1]  # diagonal through a corner
        o[6], d[6] = [c + 0.25 * w, box_hi + w, c], [0, -1, 0]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o.astype(np.float32), d.astype(np.float32)


def level_boxes(levels, roi):
    roi = np.asarray(roi, np.float64)
    c, h = (roi[:3] + roi[3:]) / 2, (roi[3:] - roi[:3]) / 2
    return [(np.float32(c - h * 2**l).astype(np.float64), np.float32(c + h * 2**l).astype(np.float64)) for l in range(levels)]


def classify(x, occ, levels, res, roi, tol=1e-3):
    """Geometric definition in fp64: returns (occupied, ambiguous) for point x:
    the finest level box holding x, the cell containing x, its bit; ambiguous
    when x lies within tol cells of a cell or box boundary."""
    boxes = level_boxes(levels, roi)
    for l, (lo, hi) in enumerate(boxes):
        u = (x - lo) / (hi - lo) * res
        if np.all((u > tol) & (u < res - tol)):
            i = np.floor(u).astype(np.int64)
            frac = u - i
            amb = bool(np.any((frac < tol) | (frac > 1 - tol)))
            return bool(occ[l * res**3 + i[0] + res * (i[1] + res * i[2])]), amb
        if np.all((u >= -tol) & (u <= res + tol)):
            return False, True  # on a box boundary
    return False, False


# ----------------------------------------------------------------------------- O2-O4 march
@pytest.mark.parametrize("levels", [1, 2, 3])
def test_all_empty_grid_emits_nothing(levels):
    rng = np.random.default_rng(2)
    o, d = random_rays(200, rng)
    occ = np.zeros(levels * 16**3, np.uint8)
    pk, t0, _, _ = O.march(occ, levels, 16, (0, 0, 0, 1, 1, 1), o, d, step=0.01)
    assert pk[:, 1].sum() == 0 and len(t0) == 0


def test_all_occupied_grid_closed_form():
    """S:248 all-ones gives the whole chord: count = #{k >= 0 : m_k in [t_enter, t_exit)}."""
    rng = np.random.default_rng(3)
    o, d = random_rays(300, rng)
    occ = np.ones(16**3, np.uint8)
    step = float(np.float32(0.0137))
    pk, t0, t1, rid = O.march(occ, 1, 16, (0, 0, 0, 1, 1, 1), o, d, step=step)
    n_amb = 0
    for r in range(len(o)):
        res = O.ray_aabb(o[r].astype(np.float64), d[r].astype(np.float64), (0, 0, 0), (1, 1, 1), 0.0, 1e10)
        if res is None:
            expect, amb = 0, False
        else:
            a = (res[0] - 0.0) / step - 0.5
            b = (res[1] - 0.0) / step - 0.5
            expect = max(0, math.ceil(b) - max(0, math.ceil(a)))
            amb = min(abs(a - round(a)), abs(b - round(b))) < 1e-3
        if amb:
            n_amb += 1
            assert abs(pk[r, 1] - expect) <= 1
        else:
            assert pk[r, 1] == expect, r
        # the emitted run is contiguous: t1_j == t0_{j+1}, t0 = fp32(k*step)
        s, c = pk[r]
        if c > 1:
            assert np.array_equal(t1[s : s + c - 1], t0[s + 1 : s + c])
        if c > 0:
            k = np.round(t0[s : s + c].astype(np.float64) / step)
            assert np.array_equal(t0[s : s + c], (k * step).astype(np.float32))
    assert n_amb <= 5


def test_lattice_values_exact_in_fp64():
    """t_k = near + k·Δt and m_k are exact in fp64 for the config steps (reading #1):
    the fp64 value equals the exact rational, so fp32 rounding happens once."""
    rng = np.random.default_rng(4)
    for step in (np.float32(1e-2), np.float32(math.sqrt(3) / 1024), np.float32(2 * math.sqrt(3) / 1024)):
        for near in (np.float32(0.0), np.float32(0.2), np.float32(0.0123)):
            for k in list(rng.integers(0, 1 << 20, 200)) + [0, 1, (1 << 20) - 1]:
                exact = Fraction(float(near)) + (int(k) + Fraction(1, 2)) * Fraction(float(step))
                fp = float(near) + (int(k) + 0.5) * float(step)
                assert Fraction(fp) == exact


def _f32_round_exact(q: Fraction) -> float:
    """Round an exact rational to the nearest fp32, ties to even -- by exact comparison with the
    two fp32 neighbours, no floating-point arithmetic (IEEE 754 roundTiesToEven)."""
    lo = float(np.float32(float(q)))  # a neighbour within one ulp
    a = np.float32(lo)
    while Fraction(float(a)) > q:
        a = np.nextafter(a, np.float32(-np.inf))
    while Fraction(float(np.nextafter(a, np.float32(np.inf)))) <= q:
        a = np.nextafter(a, np.float32(np.inf))
    b = np.nextafter(a, np.float32(np.inf))
    da, db = q - Fraction(float(a)), Fraction(float(b)) - q
    if da < db or (da == db and (int(a.view(np.uint32)) & 1) == 0):
        return float(a)
    return float(b)


def test_lattice_point_is_the_exact_value_rounded_once():
    """Reading #3: t_k and m_k are fp32(near + (k + h/2)·Δt) of the exact real, for every index the
    ABI admits (k < 2^24).  Includes k in [2^22, 2^24), where k + 1/2 is not an fp32, and anchors
    that make the fp64 sum land on an fp32 tie (a double rounding would go to even)."""
    rng = np.random.default_rng(41)
    cases = [(np.float32(2.0**-60), np.float32(2.0**-10), (1 << 23) + 2, 1),  # tie: exact rounds up
             (np.float32(-(2.0**-60)), np.float32(2.0**-10), (1 << 23) + 3, 1),  # tie: exact rounds down
             (np.float32(0.0), np.float32(2.0**-10), (1 << 23) + 2, 1)]  # a real tie: to even
    for step in (np.float32(1e-2), np.float32(math.sqrt(3) / 1024), np.float32(2.0**-10)):
        for near in (np.float32(0.0), np.float32(0.2), np.float32(1e-30), np.float32(-3.5), np.float32(2.0**-70)):
            for k in list(rng.integers(1 << 22, 1 << 24, 60)) + list(rng.integers(0, 1 << 20, 20)) + [(1 << 24) - 1]:
                cases += [(near, step, int(k), 0), (near, step, int(k), 1)]
    n_ties = 0
    for near, step, k, h in cases:
        exact = Fraction(float(near)) + (k + Fraction(h, 2)) * Fraction(float(step))
        want = _f32_round_exact(exact)
        got = O.lattice_point(near, step, k, h)
        assert got == want, (near, step, k, h, got, want)
        naive = float(np.float32(float(near) + (k + h / 2) * float(step)))
        n_ties += naive != want
    assert n_ties >= 2  # the tie cases above do defeat plain fp64 rounding


def test_far_origin_march_equals_brute_force():
    """Rays whose box crossing sits at lattice indices in [2^22, 2^24) (t ≈ 4e3-1.6e4 at Δt = 2^-10):
    the fast oracle equals the brute force over every k, with the exact midpoints above."""
    rng = np.random.default_rng(42)
    res, roi = 8, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    occ = (rng.random(res**3) < 0.4).astype(np.uint8)
    n = 24
    dist = rng.uniform(5000.0, 15000.0, n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tgt = rng.uniform(-0.4, 0.4, (n, 3))
    o = (tgt - dist[:, None] * d).astype(np.float32)
    d = d.astype(np.float32)
    for near in (0.0, float(np.float32(2.0**-60))):
        kw = dict(step=float(np.float32(2.0**-10)), near=near)
        a = O.march(occ, 1, res, roi, o, d, **kw)
        b = O.march(occ, 1, res, roi, o, d, brute=True, **kw)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert a[0][:, 1].sum() > 200


@pytest.mark.parametrize("levels,res,cone,strat", [(1, 4, 0, 0), (1, 8, 0, 1), (1, 16, 0, 0), (2, 8, 0, 0),
                                                   (3, 6, 0, 1), (1, 8, 1, 0), (3, 8, 1, 0), (2, 16, 1, 0)])
def test_fast_march_equals_brute_force(levels, res, cone, strat):
    """NS 'brute-force per-step marching on tiny grids'."""
    rng = np.random.default_rng(100 + levels * 7 + res + cone)
    o, d = random_rays(300, rng, -0.5, 0.5)
    occ = (rng.random(levels * res**3) < 0.3).astype(np.uint8)
    kw = dict(step=float(np.float32(0.021)), stratified=strat, seed=77)
    if cone:
        kw.update(cone_angle=float(np.float32(1 / 64)), max_step=float(np.float32(0.2)), near=0.05)
    a = O.march(occ, levels, res, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, **kw)
    b = O.march(occ, levels, res, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, brute=True, **kw)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert a[0][:, 1].sum() > 100


@pytest.mark.parametrize("levels,cone", [(1, 0), (3, 0), (3, 1)])
def test_emitted_midpoints_lie_in_occupied_cells(levels, cone):
    """S:369 'zero sampled midpoints fall in cells with bit 0' (exact), plus the
    converse: every lattice midpoint clearly inside an occupied cell is emitted.
    Both checked by fp64 geometry, independent of the oracle's fp32 predicate."""
    rng = np.random.default_rng(5 + levels + cone)
    res, roi = 12, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5)
    o, d = random_rays(120, rng, -0.5, 0.5)
    occ = (rng.random(levels * res**3) < 0.35).astype(np.uint8)
    step, c, near = float(np.float32(0.017)), float(np.float32(1 / 50)), float(np.float32(0.03))
    kw = dict(step=step, near=near)
    if cone:
        kw.update(cone_angle=c, max_step=1e10)
    pk, t0, t1, rid = O.march(occ, levels, res, roi, o, d, **kw)
    emitted = set()
    for j in range(len(t0)):
        m = (float(t0[j]) + float(t1[j])) / 2
        x = o[rid[j]].astype(np.float64) + m * d[rid[j]].astype(np.float64)
        occd, amb = classify(x, occ, levels, res, roi)
        assert occd or amb
        emitted.add((int(rid[j]), float(t0[j])))
    # converse on the lattice the same rule generates
    missed = 0
    for r in range(len(o)):
        t = np.float32(near)
        for _ in range(2000):
            if cone:
                dt = np.float32(min(max(np.float32(t * np.float32(c)), np.float32(step)), np.float32(1e10)))
                tn = np.float32(t + dt)
            else:
                tn = None
            if not cone:
                break
            m = (float(t) + float(tn)) / 2
            x = o[r].astype(np.float64) + m * d[r].astype(np.float64)
            occd, amb = classify(x, occ, levels, res, roi)
            if occd and not amb:
                missed += (r, float(t)) not in emitted
            t = tn
        if not cone:
            for k in range(0, 200):
                tk = float(np.float32(near + k * step))
                m = near + (k + 0.5) * step
                x = o[r].astype(np.float64) + m * d[r].astype(np.float64)
                occd, amb = classify(x, occ, levels, res, roi)
                if occd and not amb:
                    missed += (r, tk) not in emitted
    assert missed == 0


def test_cascade_with_only_level0_equals_single_grid():
    """reading #4: a point uses the finest level whose box holds it; with only
    level 0 occupied the cascade emits exactly the single-grid samples."""
    rng = np.random.default_rng(6)
    res = 8
    o, d = random_rays(200, rng, -0.5, 0.5)
    occ0 = (rng.random(res**3) < 0.4).astype(np.uint8)
    single = O.march(occ0, 1, res, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, step=0.013)
    occ3 = np.concatenate([occ0, np.zeros(2 * res**3, np.uint8)])
    casc = O.march(occ3, 3, res, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, step=0.013)
    for x, y in zip(single, casc):
        assert np.array_equal(x, y)
    # and with level 0 empty but level 1 full, no emitted midpoint lies inside box 0
    occ_b = np.concatenate([np.zeros(res**3, np.uint8), np.ones(res**3, np.uint8)])
    pk, t0, t1, rid = O.march(occ_b, 2, res, (-0.5, -0.5, -0.5, 0.5, 0.5, 0.5), o, d, step=0.013)
    m = (t0.astype(np.float64) + t1) / 2
    x = o[rid] + m[:, None] * d[rid]
    inner = np.all((x > -0.5 + 1e-5) & (x < 0.5 - 1e-5), axis=1)
    assert not inner.any()
    assert len(t0) > 0


def test_cone_lattice_is_the_stated_recurrence():
    """reading #5: dt_k = min(max(t_k c, Δt_min), Δt_max); intervals contiguous."""
    rng = np.random.default_rng(7)
    o, d = random_rays(50, rng, -2, 2)
    levels, res = 2, 8
    occ = np.ones(levels * res**3, np.uint8)
    c, dtmin, dtmax = np.float32(1 / 32), np.float32(0.01), np.float32(0.05)
    pk, t0, t1, rid = O.march(occ, levels, res, (-1, -1, -1, 1, 1, 1), o, d, near=0.1, step=float(dtmin),
                              max_step=float(dtmax), cone_angle=float(c))
    w = (t1 - t0).astype(np.float32)
    expect = np.minimum(np.maximum(t0 * c, dtmin), dtmax).astype(np.float32)
    assert np.array_equal(t1, (t0 + expect).astype(np.float32))
    assert np.all(w > 0)
    for s, n in pk:
        if n > 1:
            seg_t0, seg_t1 = t0[s : s + n], t1[s : s + n]
            assert np.all(seg_t0[1:] >= seg_t1[:-1])  # ascending, non-overlapping


def test_cfg1_sphere_closed_form():
    """CFG1: with conservative bits every lattice midpoint inside the sphere is
    emitted, so the rendered optical depth is σ0·Δt·n_in with n_in the number of
    lattice midpoints on the chord of length L = 2√(r²−b²)."""
    c = W.cfg1()
    pk, t0, t1, rid = O.march(c.occ, c.levels, c.res, c.roi, c.rays_o, c.rays_d, step=c.step)
    sig, rgb = W.field_at_intervals(W.sphere_sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
    out = O.render_fwd(pk, t0, t1, sig, rgb)
    ctr, rad, s0 = np.array([0.5, 0.5, 0.5]), 0.3, 20.0
    checked = 0
    for r in range(64):
        oo, dd = c.rays_o[r].astype(np.float64), c.rays_d[r].astype(np.float64)
        tc = np.dot(ctr - oo, dd)
        b2 = np.dot(ctr - oo, ctr - oo) - tc**2
        s, n = pk[r]
        if b2 >= rad**2:
            assert out["opacity"][r] == 0.0
            continue
        half = math.sqrt(rad**2 - b2)
        lo, hi = (tc - half) / c.step - 0.5, (tc + half) / c.step - 0.5
        if min(abs(lo - round(lo)), abs(hi - round(hi))) < 1e-3:
            continue
        n_in_expect = max(0, math.floor(hi) - max(0, math.ceil(lo)) + 1)
        mids = (t0[s : s + n].astype(np.float64) + t1[s : s + n]) / 2
        n_in = int(np.sum(np.linalg.norm(oo + mids[:, None] * dd - ctr, axis=1) <= rad))
        assert n_in == n_in_expect
        S = s0 * np.sum((t1[s : s + n].astype(np.float64) - t0[s : s + n])[np.linalg.norm(oo + mids[:, None] * dd - ctr, axis=1) <= rad])
        assert abs(out["opacity"][r] - (1 - math.exp(-S))) < 1e-12
        chord = (tc + half) - max(0.0, tc - half)  # a ray may start inside the sphere
        assert abs(S / s0 - chord) <= c.step * 1.0001
        checked += 1
    assert checked >= 20
    # the central rays saturate: T < 1e-4 well inside the sphere
    assert out["opacity"].max() > 1 - 1e-4


def test_packing_arithmetic():
    """2 rays, ray 0 yields 3 intervals, ray 1 yields 0 -> [(0,3),(3,0)];
    starts are exclusive prefix sums of counts."""
    occ = np.zeros(4**3, np.uint8)
    occ[1 + 4 * (1 + 4 * 1)] = 1  # one cell, [0.25,0.5)^3
    o = np.array([[0.0, 0.3, 0.3], [0.0, 0.9, 0.9]], np.float32)
    d = np.array([[1, 0, 0], [1, 0, 0]], np.float32)
    pk, t0, t1, rid = O.march(occ, 1, 4, (0, 0, 0, 1, 1, 1), o, d, step=float(np.float32(1 / 12)))
    assert pk.tolist() == [[0, 3], [3, 0]]
    assert rid.tolist() == [0, 0, 0]
    rng = np.random.default_rng(8)
    o2, d2 = random_rays(500, rng)
    pk2, *_ = O.march((rng.random(8**3) < 0.5).astype(np.uint8), 1, 8, (0, 0, 0, 1, 1, 1), o2, d2, step=0.01)
    assert np.array_equal(pk2[1:, 0], np.cumsum(pk2[:, 1])[:-1]) and pk2[0, 0] == 0


def test_march_deterministic_across_thread_counts():
    """identical results regardless of thread count."""
    c = W.cfg1()
    rng = np.random.default_rng(9)
    o, d = random_rays(2000, rng)
    occ = (rng.random(32**3) < 0.2).astype(np.uint8)
    O.set_num_threads(1)
    a = O.march(occ, 1, 32, c.roi, o, d, step=c.step, stratified=1, seed=5)
    O.set_num_threads(8)
    b = O.march(occ, 1, 32, c.roi, o, d, step=c.step, stratified=1, seed=5)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_stratified_anchor_within_one_step():
    """Stratified marching shifts each ray's lattice by ξ·Δt, ξ in [0,1)."""
    rng = np.random.default_rng(10)
    o, d = random_rays(300, rng)
    occ = np.ones(8**3, np.uint8)
    step = float(np.float32(0.01))
    pk, t0, t1, rid = O.march(occ, 1, 8, (0, 0, 0, 1, 1, 1), o, d, step=step, stratified=1, seed=3)
    pk0, u0, *_ = O.march(occ, 1, 8, (0, 0, 0, 1, 1, 1), o, d, step=step)
    diffs = []
    for r in range(len(o)):
        if pk[r, 1] and pk0[r, 1]:
            off = (float(t0[pk[r, 0]]) % step)
            diffs.append(off / step)
    diffs = np.array(diffs)
    assert diffs.min() >= -1e-4 and diffs.max() < 1 + 1e-4
    assert diffs.std() > 0.2  # jitter is spread over the step
