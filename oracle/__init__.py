"""CPU oracle for the NerfAcc packed-sample volume-rendering hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2305_04966_b200`` never imports it, and
this package imports nothing from the product.

The arithmetic lives in ``oracle.c`` (plain C, fp64, one sequential loop per
ray; see its header for the passage each function follows).  This module only
compiles it (``build()``) and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Grid(C.Structure):
    _fields_ = [("levels", C.c_int32), ("res", C.c_int32), ("roi", C.c_float * 6)]


class _March(C.Structure):
    _fields_ = [
        ("near_plane", C.c_float),
        ("far_plane", C.c_float),
        ("step", C.c_float),
        ("max_step", C.c_float),
        ("cone_angle", C.c_float),
        ("stratified", C.c_int32),
        ("seed", C.c_uint64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_u24.restype = C.c_double
        _lib.or_contract.restype = C.c_double
        _lib.or_contract.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        _lib.or_uncontract.restype = C.c_double
        _lib.or_uncontract.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        _lib.or_field_sigma.restype = C.c_double
        _lib.or_field_sigma.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_void_p]
        _lib.or_num_threads.restype = C.c_int
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    """fp32 GPU-side arrays are widened exactly to fp64."""
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def set_num_threads(n: int) -> None:
    lib().or_set_num_threads(int(n))


def _i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


def num_threads() -> int:
    return lib().or_num_threads()


# --------------------------------------------------------------------------- RNG
def philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(x) for x in o]


# --------------------------------------------------------------------------- geometry
def lattice_point(near, step, k, half):
    f = lib().or_lattice_point
    f.restype = C.c_float
    f.argtypes = [C.c_float, C.c_float, C.c_int64, C.c_int32]
    return float(f(float(near), float(step), int(k), int(half)))


def ray_aabb(o, d, lo, hi, near=0.0, far=np.inf):
    """O1 slab test; returns (t_enter, t_exit) or None."""
    arr = lambda v: (C.c_double * 3)(*[float(x) for x in v])
    te, tx = C.c_double(), C.c_double()
    ok = lib().or_ray_aabb(arr(o), arr(d), arr(lo), arr(hi), C.c_double(near), C.c_double(far),
                           C.byref(te), C.byref(tx))
    return (te.value, tx.value) if ok else None


def contract(map_kind: int, s: float, tn: float, tf: float) -> float:
    return lib().or_contract(map_kind, s, tn, tf)


def uncontract(map_kind: int, t: float, tn: float, tf: float) -> float:
    return lib().or_uncontract(map_kind, t, tn, tf)


# --------------------------------------------------------------------------- march
def _grid(levels, res, roi):
    g = _Grid()
    g.levels, g.res = int(levels), int(res)
    for i in range(6):
        g.roi[i] = float(roi[i])
    return g


def _march(near, far, step, max_step=1e10, cone_angle=0.0, stratified=0, seed=0):
    p = _March()
    p.near_plane, p.far_plane, p.step = near, far, step
    p.max_step, p.cone_angle, p.stratified, p.seed = max_step, cone_angle, int(stratified), int(seed)
    return p


def march(occ, levels, res, roi, rays_o, rays_d, *, near=0.0, far=1e10, step, max_step=1e10,
          cone_angle=0.0, stratified=0, seed=0, t_min=None, t_max=None, brute=False):
    """O2-O4: packed occupancy-grid marching.  occ is uint8 [levels*res^3]
    (x fastest).  Returns (packed_info int64 [n,2], t0 f32, t1 f32, ray_id i32)."""
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    assert occ.size == levels * res ** 3
    o, d = _f32(rays_o).reshape(-1, 3), _f32(rays_d).reshape(-1, 3)
    n = o.shape[0]
    t_min, t_max = _f32(t_min), _f32(t_max)
    g, p = _grid(levels, res, roi), _march(near, far, step, max_step, cone_angle, stratified, seed)
    counts = np.zeros(n, np.int64)
    lib().or_march_count(C.byref(g), _p(occ), C.byref(p), _p(o), _p(d), _p(t_min), _p(t_max),
                         C.c_int64(n), C.c_int(int(brute)), _p(counts))
    start = np.zeros(n, np.int64)
    if n:
        start[1:] = np.cumsum(counts)[:-1]
    total = int(counts.sum())
    t0 = np.empty(total, np.float32)
    t1 = np.empty(total, np.float32)
    rid = np.empty(total, np.int32)
    lib().or_march_fill(C.byref(g), _p(occ), C.byref(p), _p(o), _p(d), _p(t_min), _p(t_max),
                        C.c_int64(n), C.c_int(int(brute)), _p(start), _p(t0), _p(t1), _p(rid))
    packed = np.stack([start, counts], axis=1)
    return packed, t0, t1, rid


def march_counts(occ, levels, res, roi, rays_o, rays_d, *, near=0.0, far=1e10, step,
                 max_step=1e10, cone_angle=0.0, stratified=0, seed=0, t_min=None, t_max=None,
                 brute=False):
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    o, d = _f32(rays_o).reshape(-1, 3), _f32(rays_d).reshape(-1, 3)
    n = o.shape[0]
    g, p = _grid(levels, res, roi), _march(near, far, step, max_step, cone_angle, stratified, seed)
    counts = np.zeros(n, np.int64)
    lib().or_march_count(C.byref(g), _p(occ), C.byref(p), _p(o), _p(d), _p(_f32(t_min)),
                         _p(_f32(t_max)), C.c_int64(n), C.c_int(int(brute)), _p(counts))
    return counts


# --------------------------------------------------------------------------- filter
def filter_counts(packed_info, t0, t1, sigma, neg_log_eps):
    """O5: kept prefix length per ray and the decision margin min |S_i - L_eps|."""
    pi = _i64(packed_info).reshape(-1, 2)
    n = pi.shape[0]
    cnt = np.zeros(n, np.int64)
    margin = np.zeros(n, np.float64)
    lib().or_filter_cut(_p(pi), C.c_int64(n), _p(_f64(t0)), _p(_f64(t1)), _p(_f64(sigma)),
                        C.c_double(neg_log_eps), _p(cnt), _p(margin))
    return cnt, margin


def filter_early_stop(packed_info, t0, t1, sigma, neg_log_eps):
    """O5 + compaction: returns (packed_info', t0', t1', ray_id', margin)."""
    pi = _i64(packed_info).reshape(-1, 2)
    cnt, margin = filter_counts(pi, t0, t1, sigma, neg_log_eps)
    start = np.zeros_like(cnt)
    if cnt.size:
        start[1:] = np.cumsum(cnt)[:-1]
    idx = np.concatenate([np.arange(s, s + c) for (s, _), c in zip(pi, cnt)]) if cnt.sum() else np.zeros(0, np.int64)
    rid = np.repeat(np.arange(pi.shape[0], dtype=np.int32), cnt)
    return np.stack([start, cnt], 1), np.asarray(t0)[idx], np.asarray(t1)[idx], rid, margin


# --------------------------------------------------------------------------- render
def render_fwd(packed_info, t0, t1, sigma, rgb=None, neg_log_eps=np.inf):
    """O6.  Returns dict(trans, alphas, weights, color, opacity, depth) in fp64."""
    pi = _i64(packed_info).reshape(-1, 2)
    n, N = pi.shape[0], len(t0)
    out = {k: np.zeros(N) for k in ("trans", "alphas", "weights")}
    out["color"] = np.zeros((n, 3))
    out["opacity"] = np.zeros(n)
    out["depth"] = np.zeros(n)
    rgbf = None if rgb is None else _f64(rgb).reshape(-1, 3)
    lib().or_render_fwd(_p(pi), C.c_int64(n), _p(_f64(t0)), _p(_f64(t1)), _p(_f64(sigma)), _p(rgbf),
                        C.c_double(neg_log_eps), _p(out["trans"]), _p(out["alphas"]),
                        _p(out["weights"]), _p(out["color"]), _p(out["opacity"]), _p(out["depth"]))
    return out


def render_bwd(packed_info, t0, t1, sigma, rgb, g_color=None, g_opacity=None, g_depth=None,
               neg_log_eps=np.inf):
    """O7.  Returns (g_sigma [N], g_rgb [N,3]) in fp64."""
    pi = _i64(packed_info).reshape(-1, 2)
    n, N = pi.shape[0], len(t0)
    gs, grgb = np.zeros(N), np.zeros((N, 3))
    lib().or_render_bwd(_p(pi), C.c_int64(n), _p(_f64(t0)), _p(_f64(t1)), _p(_f64(sigma)),
                        _p(_f64(rgb).reshape(-1, 3)), C.c_double(neg_log_eps),
                        _p(_f64(g_color)), _p(_f64(g_opacity)), _p(_f64(g_depth)), _p(gs), _p(grgb))
    return gs, grgb


def weights_bwd(packed_info, t0, t1, sigma, g_weights, g_trans=None, neg_log_eps=np.inf):
    pi = _i64(packed_info).reshape(-1, 2)
    gs = np.zeros(len(t0))
    lib().or_weights_bwd(_p(pi), C.c_int64(pi.shape[0]), _p(_f64(t0)), _p(_f64(t1)),
                         _p(_f64(sigma)), C.c_double(neg_log_eps), _p(_f64(g_weights)),
                         _p(_f64(g_trans)), _p(gs))
    return gs


def weights_alpha_fwd(packed_info, alpha, neg_log_eps=np.inf):
    """Alpha compositing (oracle.h or_weights_alpha_fwd): returns (w, T)."""
    pi = _i64(packed_info).reshape(-1, 2)
    w = np.zeros(len(alpha))
    T = np.zeros(len(alpha))
    lib().or_weights_alpha_fwd(_p(pi), C.c_int64(pi.shape[0]), _p(_f64(alpha)), C.c_double(neg_log_eps), _p(w),
                               _p(T))
    return w, T


def weights_alpha_bwd(packed_info, alpha, g_weights, g_trans=None, neg_log_eps=np.inf):
    pi = _i64(packed_info).reshape(-1, 2)
    ga = np.zeros(len(alpha))
    lib().or_weights_alpha_bwd(_p(pi), C.c_int64(pi.shape[0]), _p(_f64(alpha)), C.c_double(neg_log_eps),
                               _p(_f64(g_weights)), _p(_f64(g_trans)), _p(ga))
    return ga


def accumulate(packed_info, weights, values=None, C_=1):
    pi = _i64(packed_info).reshape(-1, 2)
    n = pi.shape[0]
    if values is not None:
        values = _f64(values)
        values = values.reshape(len(weights), -1) if values.ndim != 2 else values
        C_ = values.shape[1]
    out = np.zeros((n, C_))
    lib().or_accumulate(_p(pi), C.c_int64(n), _p(_f64(weights)), _p(values), C.c_int32(C_), _p(out))
    return out


def accumulate_bwd(packed_info, weights, values, g_out):
    pi = _i64(packed_info).reshape(-1, 2)
    n = pi.shape[0]
    g_out = _f64(g_out).reshape(n, -1)
    C_ = g_out.shape[1]
    if values is not None:
        values = _f64(values).reshape(len(weights), C_)
    gw = np.zeros(len(weights))
    gv = np.zeros((len(weights), C_)) if values is not None else None
    lib().or_accumulate_bwd(_p(pi), C.c_int64(n), _p(_f64(weights)), _p(values), C.c_int32(C_),
                            _p(g_out), _p(gw), _p(gv))
    return gw, gv


# --------------------------------------------------------------------------- resample
def importance_sample(s_edges, n_out, *, sigma=None, cdf=None, map_kind=1, t_near=0.2,
                      t_far=1000.0, stratified=0, seed=0, want_t=True):
    """O8.  s_edges [n_rays, n_in+1]; returns (s_out, t_out) fp64 [n_rays, n_out+1]."""
    e = _f64(s_edges)
    n, n_in = e.shape[0], e.shape[1] - 1
    assert (sigma is None) != (cdf is None)
    s_out = np.zeros((n, n_out + 1))
    t_out = np.zeros((n, n_out + 1)) if want_t else None
    lib().or_importance_sample(C.c_int64(n), C.c_int32(n_in), _p(e), _p(_f64(sigma)), _p(_f64(cdf)),
                               C.c_int(map_kind), C.c_double(t_near), C.c_double(t_far),
                               C.c_int32(n_out), C.c_int32(stratified), C.c_uint64(seed),
                               _p(s_out), _p(t_out))
    return s_out, t_out


def importance_sample_ranged(s_edges, n_out, t_near, t_far, *, sigma=None, cdf=None, map_kind=1, stratified=0,
                             seed=0, want_t=True):
    """O8 with per-ray [t_near, t_far] arrays (combined estimator, reading #19)."""
    e = _f64(s_edges)
    n, n_in = e.shape[0], e.shape[1] - 1
    assert (sigma is None) != (cdf is None)
    s_out = np.zeros((n, n_out + 1))
    t_out = np.zeros((n, n_out + 1)) if want_t else None
    lib().or_importance_sample_ranged(C.c_int64(n), C.c_int32(n_in), _p(e), _p(_f64(sigma)), _p(_f64(cdf)),
                                      C.c_int(map_kind), _p(_f64(t_near)), _p(_f64(t_far)), C.c_int32(n_out),
                                      C.c_int32(stratified), C.c_uint64(seed), _p(s_out), _p(t_out))
    return s_out, t_out


def ray_bounds(occ, levels, res, roi, rays_o, rays_d, *, near=0.0, far=1e10, step, max_step=1e10,
               cone_angle=0.0, stratified=0, seed=0, t_min=None, t_max=None):
    """Combined estimator, grid stage (reading #18): per-ray (t_near, t_far) f32 of the
    intervals march() emits; (0, 0) for rays it culls."""
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    o, d = _f32(rays_o).reshape(-1, 3), _f32(rays_d).reshape(-1, 3)
    n = o.shape[0]
    t_min, t_max = _f32(t_min), _f32(t_max)
    g, p = _grid(levels, res, roi), _march(near, far, step, max_step, cone_angle, stratified, seed)
    tn = np.zeros(n, np.float32)
    tf = np.zeros(n, np.float32)
    lib().or_ray_bounds(C.byref(g), _p(occ), C.byref(p), _p(o), _p(d), _p(t_min), _p(t_max), C.c_int64(n),
                        _p(tn), _p(tf))
    return tn, tf


def importance_cdf(s_edges, *, sigma=None, cdf=None, map_kind=1, t_near=0.2, t_far=1000.0):
    e = _f64(s_edges)
    n, n_in = e.shape[0], e.shape[1] - 1
    F = np.zeros((n, n_in + 1))
    lib().or_importance_cdf(C.c_int64(n), C.c_int32(n_in), _p(e), _p(_f64(sigma)), _p(_f64(cdf)),
                            C.c_int(map_kind), C.c_double(t_near), C.c_double(t_far), _p(F))
    return F


def pdf_loss(t, w, th, wh, eps=1e-7):
    """Proposal supervision loss per ray (reading #21): t [n, nf+1], w [n, nf], th [n, np+1], wh [n, np]."""
    t, w, th, wh = (np.ascontiguousarray(x, np.float64) for x in (t, w, th, wh))
    n, nf, np_ = t.shape[0], w.shape[1], wh.shape[1]
    loss = np.zeros(n)
    lib().or_pdf_loss(C.c_int64(n), C.c_int32(nf), _p(t), _p(w), C.c_int32(np_), _p(th), _p(wh), C.c_double(eps),
                      _p(loss))
    return loss


def pdf_loss_bwd(t, w, th, wh, g_loss, eps=1e-7):
    t, w, th, wh = (np.ascontiguousarray(x, np.float64) for x in (t, w, th, wh))
    n, nf, np_ = t.shape[0], w.shape[1], wh.shape[1]
    g = np.zeros((n, np_))
    lib().or_pdf_loss_bwd(C.c_int64(n), C.c_int32(nf), _p(t), _p(w), C.c_int32(np_), _p(th), _p(wh),
                          C.c_double(eps), _p(_f64(g_loss)), _p(g))
    return g


# --------------------------------------------------------------------------- grid update
def occgrid_points(levels, res, roi, seed, step, jitter, cell_begin=0, cell_count=None):
    g = _grid(levels, res, roi)
    if cell_count is None:
        cell_count = levels * res ** 3 - cell_begin
    xyz = np.zeros((cell_count, 3), np.float32)
    lib().or_occgrid_points(C.byref(g), C.c_uint64(seed), C.c_int64(step), C.c_int32(jitter),
                            C.c_int64(cell_begin), C.c_int64(cell_count), _p(xyz))
    return xyz


def occgrid_times(levels, res, roi, seed, step, draw, cell_begin=0, cell_count=None):
    """Per-cell timestamps of draw `draw` for dynamic scenes (reading #20)."""
    g = _grid(levels, res, roi)
    if cell_count is None:
        cell_count = levels * res ** 3 - cell_begin
    t = np.zeros(cell_count, np.float32)
    lib().or_occgrid_times(C.byref(g), C.c_uint64(seed), C.c_int64(step), C.c_int32(draw), C.c_int64(cell_begin),
                           C.c_int64(cell_count), _p(t))
    return t


def occgrid_update(levels, res, roi, density, fresh, *, rule=0, decay=0.95, threshold=0.01,
                   thresh_rule=0):
    """O9.  Returns (density' f32, bits uint8, mean)."""
    g = _grid(levels, res, roi)
    dens = np.array(density, dtype=np.float32, copy=True).ravel()
    bits = np.zeros(dens.size, np.uint8)
    mean = C.c_double()
    lib().or_occgrid_update(C.byref(g), _p(dens), _p(_f32(fresh).ravel()), C.c_int32(rule),
                            C.c_float(decay), C.c_float(threshold), C.c_int32(thresh_rule),
                            _p(bits), C.byref(mean))
    return dens, bits, mean.value


# --------------------------------------------------------------------------- validation fields
def field_sigma(kind, params, sigma0, x):
    prm = (C.c_double * len(params))(*params)
    xx = (C.c_double * 3)(*[float(v) for v in x])
    return lib().or_field_sigma(kind, prm, C.c_double(sigma0), xx)


def render_quadrature(kind, params, sigma0, o, d, t_a, t_b, n_quad):
    prm = (C.c_double * len(params))(*params)
    arr = lambda v: (C.c_double * 3)(*[float(x) for x in v])
    op, dp = C.c_double(), C.c_double()
    lib().or_render_quadrature(kind, prm, C.c_double(sigma0), arr(o), arr(d), C.c_double(t_a),
                               C.c_double(t_b), C.c_int64(n_quad), C.byref(op), C.byref(dp))
    return op.value, dp.value
