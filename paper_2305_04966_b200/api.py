"""Thin PyTorch binding of libnacc (include/nacc.h), named after Algorithm 1
of the paper.  Argument marshalling only: every step of the path
runs in the library's CUDA kernels; torch provides device memory, streams and
the process group.  Non-CUDA tensors are rejected (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import Callable, Optional

import torch

from . import _lib as L
from ._lib import check

NEG_LOG_EPS_DEFAULT = -math.log(float(torch.tensor(1e-4, dtype=torch.float32)))  # P:86, ε = 1e-4 (fp32)


def neg_log_eps(eps: Optional[float]) -> float:
    """-ln ε in fp64 on the host (reading #9); None or 0 disables early stop."""
    if eps is None or eps <= 0.0:
        return math.inf
    return -math.log(float(torch.tensor(eps, dtype=torch.float32)))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _req(t: torch.Tensor, dtype, name: str, numel: Optional[int] = None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        t = t.contiguous()
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    return t


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


# ----------------------------------------------------------------------------- specs
@dataclasses.dataclass
class GridSpec:
    """Occupancy grid: `levels` cascaded boxes centre ± half·2^l of
    `roi`, `res`^3 cells each (reading #4)."""
    roi: tuple = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    res: int = 128
    levels: int = 1

    def c(self) -> L.Grid:
        g = L.Grid()
        g.levels, g.res = int(self.levels), int(self.res)
        for i in range(6):
            g.roi[i] = float(self.roi[i])
        return g

    @property
    def n_cells(self) -> int:
        return self.levels * self.res ** 3


@dataclasses.dataclass
class MarchParams:
    """Ray-marching parameters (readings #1, #5)."""
    step: float
    near_plane: float = 0.0
    far_plane: float = 1e10
    max_step: float = 1e10
    cone_angle: float = 0.0
    stratified: bool = False
    seed: int = 0

    def c(self) -> L.March:
        m = L.March()
        m.near_plane, m.far_plane, m.step = self.near_plane, self.far_plane, self.step
        m.max_step, m.cone_angle = self.max_step, self.cone_angle
        m.stratified, m.seed = int(bool(self.stratified)), int(self.seed)
        return m


@dataclasses.dataclass
class PackedSamples:
    """Sample-as-interval packed tensor: t0, t1 fp32 [N], ray_id
    int32 [N], packed_info int64 [n_rays, 2] = (start, count).

    In device-count mode (``sync=False``) the arrays have a fixed capacity,
    ``total`` (device int64 [1]) holds N and nothing waits for the host, so a
    whole step can be captured in a CUDA graph."""
    packed_info: torch.Tensor
    t0: torch.Tensor
    t1: torch.Tensor
    ray_id: torch.Tensor
    total: Optional[torch.Tensor] = None
    status: Optional[torch.Tensor] = None

    @property
    def n_rays(self) -> int:
        return self.packed_info.shape[0]

    @property
    def n_samples(self) -> int:
        """N when synced; the capacity in device-count mode."""
        return self.t0.numel()


# ----------------------------------------------------------------------------- sampling
def prepare_bits(grid: GridSpec, fine_bits: torch.Tensor) -> torch.Tensor:
    """A full bitfield buffer (public fine bits + the library's skip mask) from
    fine bits packed as in nacc.h; ``OccupancyGrid.bits`` is already prepared."""
    g = grid.c()
    nb = L.lib().nacc_grid_bits_bytes(C.byref(g)) // 4
    fine_bits = _req(fine_bits, torch.int32, "bits")
    full = torch.zeros(nb, dtype=torch.int32, device=fine_bits.device)
    n = min(fine_bits.numel(), nb)
    full[:n] = fine_bits.reshape(-1)[:n]
    check(L.lib().nacc_grid_prepare(C.byref(g), _ptr(full), _stream()), "nacc_grid_prepare")
    return full


def sampling_occgrid(rays_o: torch.Tensor, rays_d: torch.Tensor, grid: GridSpec, bits: torch.Tensor,
                     params: MarchParams, t_min: Optional[torch.Tensor] = None,
                     t_max: Optional[torch.Tensor] = None, capacity: Optional[int] = None,
                     sync: bool = True) -> PackedSamples:
    """Alg. 1 ``nerfacc.sampling`` with the occupancy-grid estimator.
    ``capacity`` enables the one-shot single-pass march; without it the exact
    path runs (count + scan, read the total, fill).  ``sync=False`` (needs a
    capacity) returns capacity-sized arrays with a device total and a device
    status (NACC_ERR_INSUFFICIENT_CAPACITY if the capacity was too small)."""
    lib = L.lib()
    n = rays_o.shape[0]
    dev = rays_o.device
    rays_o = _req(rays_o, torch.float32, "rays_o", 3 * n)
    rays_d = _req(rays_d, torch.float32, "rays_d", 3 * n)
    bits = _req(bits, torch.int32, "bits")
    if bits.numel() * 4 < lib.nacc_grid_bits_bytes(C.byref(grid.c())):
        raise ValueError("bits must be a full prepared bitfield (OccupancyGrid.bits or prepare_bits())")
    if t_min is not None:
        t_min = _req(t_min, torch.float32, "t_min", n)
    if t_max is not None:
        t_max = _req(t_max, torch.float32, "t_max", n)
    g, p = grid.c(), params.c()
    ws = _ws(lib.nacc_sampling_occgrid_workspace_bytes(C.byref(g), C.byref(p), n), dev)
    packed = torch.empty((n, 2), dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)  # always written by the call
    cap = int(capacity) if capacity is not None else 0
    t0 = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    t1 = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    rid = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    with_out = cap > 0
    status = torch.empty(1, dtype=torch.int32, device=dev)
    check(lib.nacc_sampling_occgrid(C.byref(g), _ptr(bits), C.byref(p), _ptr(rays_o), _ptr(rays_d), _ptr(t_min),
                                    _ptr(t_max), n, _ptr(packed), _ptr(t0) if with_out else None,
                                    _ptr(t1) if with_out else None, _ptr(rid) if with_out else None, cap,
                                    _ptr(total), _ptr(status), _ptr(ws), ws.numel(), _stream()),
          "nacc_sampling_occgrid")
    if not sync:
        if not with_out:
            raise ValueError("sync=False needs a capacity")
        return PackedSamples(packed, t0, t1, rid, total, status)
    N = int(total.item())
    st = int(status.item())
    if st not in (L.NACC_OK, L.NACC_ERR_INSUFFICIENT_CAPACITY):
        # e.g. the shared cone lattice overflowed its 2^20-entry table: the samples would be truncated
        raise L.NaccError(st, "nacc_sampling_occgrid: device status (the shared cone lattice is longer than "
                              "2^20 intervals: raise step or cone_angle, or lower far_plane)")
    if N > cap:
        t0 = torch.empty(max(N, 1), dtype=torch.float32, device=dev)
        t1 = torch.empty(max(N, 1), dtype=torch.float32, device=dev)
        rid = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
        check(lib.nacc_sampling_occgrid_fill(C.byref(g), _ptr(bits), C.byref(p), _ptr(rays_o), _ptr(rays_d),
                                             _ptr(t_min), _ptr(t_max), n, _ptr(packed), _ptr(t0), _ptr(t1),
                                             _ptr(rid), _ptr(ws), ws.numel(), _stream()),
              "nacc_sampling_occgrid_fill")
    return PackedSamples(packed, t0[:N], t1[:N], rid[:N])


def filter_early_stop(samples: PackedSamples, sigma: torch.Tensor, eps: Optional[float] = 1e-4,
                      sync: bool = True) -> PackedSamples:
    """§4.2 no-gradient filtering: keep each ray's prefix with entering
    transmittance >= ε.  ``sigma`` comes from the caller's no-grad density query.
    ``sync=False`` keeps the input capacity and returns a device total."""
    lib = L.lib()
    n, N = samples.n_rays, samples.n_samples
    dev = samples.packed_info.device
    sigma = _req(sigma.detach(), torch.float32, "sigma", N)
    ws = _ws(lib.nacc_filter_workspace_bytes(n), dev)
    packed = torch.empty((n, 2), dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)  # always written by the call
    cap = max(N, 1)
    t0 = torch.empty(cap, dtype=torch.float32, device=dev)
    t1 = torch.empty(cap, dtype=torch.float32, device=dev)
    rid = torch.empty(cap, dtype=torch.int32, device=dev)
    check(lib.nacc_filter_early_stop(_ptr(samples.packed_info), n, _ptr(samples.t0), _ptr(samples.t1), _ptr(sigma),
                                     N, neg_log_eps(eps), _ptr(packed), _ptr(t0), _ptr(t1), _ptr(rid), cap,
                                     _ptr(total), _ptr(ws), ws.numel(), _stream()), "nacc_filter_early_stop")
    if not sync:
        return PackedSamples(packed, t0, t1, rid, total)
    M = int(total.item())
    return PackedSamples(packed, t0[:M], t1[:M], rid[:M])


# ----------------------------------------------------------------------------- rendering
class _RenderFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, packed_info, ray_id, t0, t1, sigma, rgb, nle):
        n, N = packed_info.shape[0], t0.numel()
        dev = t0.device
        color = torch.empty((n, 3), dtype=torch.float32, device=dev)
        opacity = torch.empty(n, dtype=torch.float32, device=dev)
        depth = torch.empty(n, dtype=torch.float32, device=dev)
        cx = torch.empty((n, 5), dtype=torch.float64, device=dev)
        check(L.lib().nacc_render_fwd(_ptr(packed_info), _ptr(ray_id), n, _ptr(t0), _ptr(t1), _ptr(sigma), _ptr(rgb),
                                      N, nle, _ptr(color), _ptr(opacity), _ptr(depth), _ptr(cx), _stream()),
              "nacc_render_fwd")
        ctx.save_for_backward(packed_info, ray_id, t0, t1, sigma, rgb, cx)
        ctx.nle = nle
        ctx.set_materialize_grads(False)  # unused outputs pass NULL gradients, not zero tensors
        return color, opacity, depth

    @staticmethod
    def backward(ctx, g_color, g_opacity, g_depth):
        packed_info, ray_id, t0, t1, sigma, rgb, cx = ctx.saved_tensors
        n, N = packed_info.shape[0], t0.numel()
        g_sigma = torch.empty_like(sigma)
        g_rgb = torch.empty_like(rgb)
        gc = None if g_color is None else g_color.contiguous().float()
        go = None if g_opacity is None else g_opacity.contiguous().float()
        gd = None if g_depth is None else g_depth.contiguous().float()
        ws = _ws(L.lib().nacc_render_bwd_workspace_bytes(n), t0.device)
        check(L.lib().nacc_render_bwd(_ptr(packed_info), _ptr(ray_id), n, _ptr(t0), _ptr(t1), _ptr(sigma), _ptr(rgb),
                                      N, ctx.nle, _ptr(cx), _ptr(gc), _ptr(go), _ptr(gd), _ptr(g_sigma),
                                      _ptr(g_rgb), _ptr(ws), ws.numel(), _stream()), "nacc_render_bwd")
        return None, None, None, None, g_sigma, g_rgb, None


def rendering(samples: PackedSamples, sigma: torch.Tensor, rgb: torch.Tensor, eps: Optional[float] = None):
    """Alg. 1 ``nerfacc.rendering`` on caller-evaluated σ and rgb:
    returns (color [n,3], opacity [n], depth [n]), differentiable w.r.t. σ and rgb."""
    N = samples.n_samples
    sigma = _req(sigma, torch.float32, "sigma", N)
    rgb = _req(rgb, torch.float32, "rgb", 3 * N)
    rid = samples.ray_id if samples.ray_id.numel() == N else None
    return _RenderFn.apply(samples.packed_info, rid, samples.t0, samples.t1, sigma, rgb.view(N, 3), neg_log_eps(eps))


def render_fwd(samples: PackedSamples, sigma: torch.Tensor, rgb: torch.Tensor, eps: Optional[float] = None):
    """Functional (no autograd) ``nacc_render_fwd``: returns (color, opacity,
    depth, ctx).  Works in device-count mode (no host sync; graph-capturable)."""
    n, N = samples.n_rays, samples.n_samples
    dev = samples.t0.device
    sigma = _req(sigma.detach(), torch.float32, "sigma", N)
    rgb = _req(rgb.detach(), torch.float32, "rgb", 3 * N)
    color = torch.empty((n, 3), dtype=torch.float32, device=dev)
    opacity = torch.empty(n, dtype=torch.float32, device=dev)
    depth = torch.empty(n, dtype=torch.float32, device=dev)
    cx = torch.empty((n, 5), dtype=torch.float64, device=dev)
    check(L.lib().nacc_render_fwd(_ptr(samples.packed_info), _ptr(samples.ray_id), n, _ptr(samples.t0),
                                  _ptr(samples.t1), _ptr(sigma), _ptr(rgb), N, neg_log_eps(eps), _ptr(color),
                                  _ptr(opacity), _ptr(depth), _ptr(cx), _stream()), "nacc_render_fwd")
    return color, opacity, depth, cx


def render_bwd(samples: PackedSamples, sigma: torch.Tensor, rgb: torch.Tensor, ctx: torch.Tensor,
               g_color: Optional[torch.Tensor] = None, g_opacity: Optional[torch.Tensor] = None,
               g_depth: Optional[torch.Tensor] = None, eps: Optional[float] = None):
    """Functional ``nacc_render_bwd``: returns (g_sigma, g_rgb)."""
    n, N = samples.n_rays, samples.n_samples
    sigma = _req(sigma.detach(), torch.float32, "sigma", N)
    rgb = _req(rgb.detach(), torch.float32, "rgb", 3 * N)
    g_sigma = torch.empty_like(sigma)
    g_rgb = torch.empty_like(rgb)
    ws = _ws(L.lib().nacc_render_bwd_workspace_bytes(n), samples.t0.device)
    check(L.lib().nacc_render_bwd(_ptr(samples.packed_info), _ptr(samples.ray_id), n, _ptr(samples.t0),
                                  _ptr(samples.t1), _ptr(sigma), _ptr(rgb), N, neg_log_eps(eps), _ptr(ctx),
                                  _ptr(g_color), _ptr(g_opacity), _ptr(g_depth), _ptr(g_sigma), _ptr(g_rgb),
                                  _ptr(ws), ws.numel(), _stream()), "nacc_render_bwd")
    return g_sigma, g_rgb


class _WeightsFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, packed_info, t0, t1, sigma, nle, ray_id):
        n, N = packed_info.shape[0], t0.numel()
        w = torch.empty_like(sigma)
        T = torch.empty_like(sigma)
        a = torch.empty_like(sigma)
        if ray_id is not None:  # samples from the sampling calls: the flat-tile kernel
            check(L.lib().nacc_render_weights_fwd_flat(_ptr(packed_info), _ptr(ray_id), n, _ptr(t0), _ptr(t1),
                                                       _ptr(sigma), N, nle, _ptr(w), _ptr(T), _ptr(a), _stream()),
                  "nacc_render_weights_fwd_flat")
        else:
            check(L.lib().nacc_render_weights_fwd(_ptr(packed_info), n, _ptr(t0), _ptr(t1), _ptr(sigma), N, nle,
                                                  _ptr(w), _ptr(T), _ptr(a), _stream()), "nacc_render_weights_fwd")
        ctx.save_for_backward(packed_info, t0, t1, sigma, ray_id)
        ctx.nle = nle
        ctx.mark_non_differentiable(a)
        return w, T, a

    @staticmethod
    def backward(ctx, g_w, g_T, g_a):
        packed_info, t0, t1, sigma, ray_id = ctx.saved_tensors
        n, N = packed_info.shape[0], t0.numel()
        g_sigma = torch.empty_like(sigma)
        gw = torch.zeros_like(sigma) if g_w is None else g_w.contiguous().float()
        gT = None if g_T is None else g_T.contiguous().float()
        if ray_id is not None:  # the flat-tile backward (per-ray totals in a workspace)
            ws = _ws(L.lib().nacc_render_weights_bwd_flat_workspace_bytes(n), t0.device)
            check(L.lib().nacc_render_weights_bwd_flat(_ptr(packed_info), _ptr(ray_id), n, _ptr(t0), _ptr(t1),
                                                       _ptr(sigma), N, ctx.nle, _ptr(gw), _ptr(gT), _ptr(g_sigma),
                                                       _ptr(ws), ws.numel(), _stream()), "nacc_render_weights_bwd_flat")
        else:
            check(L.lib().nacc_render_weights_bwd(_ptr(packed_info), n, _ptr(t0), _ptr(t1), _ptr(sigma), N, ctx.nle,
                                                  _ptr(gw), _ptr(gT), _ptr(g_sigma), _stream()),
                  "nacc_render_weights_bwd")
        return None, None, None, g_sigma, None, None


def render_weights(samples: PackedSamples, sigma: torch.Tensor, eps: Optional[float] = None):
    """Transmittance estimator (Eq. 2): returns (weights, trans, alphas) per sample.  Samples
    carrying ray_id (the sampling calls' output: contiguous packing) take the flat-tile forward;
    a PackedSamples with an empty ray_id takes the one-warp-per-ray kernel (any packing)."""
    sigma = _req(sigma, torch.float32, "sigma", samples.n_samples)
    rid = samples.ray_id if samples.ray_id is not None and samples.ray_id.numel() == samples.n_samples else None
    return _WeightsFn.apply(samples.packed_info, samples.t0, samples.t1, sigma, neg_log_eps(eps), rid)


class _AlphaWeightsFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, packed_info, alphas, nle, ray_id):
        n, N = packed_info.shape[0], alphas.numel()
        w = torch.empty_like(alphas)
        T = torch.empty_like(alphas)
        if ray_id is not None:  # samples from the sampling calls: the flat-tile kernel
            check(L.lib().nacc_render_weights_alpha_fwd_flat(_ptr(packed_info), _ptr(ray_id), n, _ptr(alphas), N, nle,
                                                             _ptr(w), _ptr(T), _stream()),
                  "nacc_render_weights_alpha_fwd_flat")
        else:
            check(L.lib().nacc_render_weights_alpha_fwd(_ptr(packed_info), n, _ptr(alphas), N, nle, _ptr(w), _ptr(T),
                                                        _stream()), "nacc_render_weights_alpha_fwd")
        ctx.save_for_backward(packed_info, alphas, ray_id)
        ctx.nle = nle
        ctx.set_materialize_grads(False)
        return w, T

    @staticmethod
    def backward(ctx, g_w, g_T):
        packed_info, alphas, ray_id = ctx.saved_tensors
        n, N = packed_info.shape[0], alphas.numel()
        g_a = torch.empty_like(alphas)
        gw = torch.zeros_like(alphas) if g_w is None else g_w.contiguous().float()
        gT = None if g_T is None else g_T.contiguous().float()
        ws = _ws(L.lib().nacc_render_weights_alpha_bwd_workspace_bytes(N), alphas.device)
        if ray_id is not None:  # the flat-tile backward
            check(L.lib().nacc_render_weights_alpha_bwd_flat(_ptr(packed_info), _ptr(ray_id), n, _ptr(alphas), N,
                                                             ctx.nle, _ptr(gw), _ptr(gT), _ptr(g_a), _ptr(ws),
                                                             ws.numel(), _stream()), "nacc_render_weights_alpha_bwd_flat")
        else:
            check(L.lib().nacc_render_weights_alpha_bwd(_ptr(packed_info), n, _ptr(alphas), N, ctx.nle, _ptr(gw),
                                                        _ptr(gT), _ptr(g_a), _ptr(ws), ws.numel(), _stream()),
                  "nacc_render_weights_alpha_bwd")
        return None, g_a, None, None


def render_weights_alpha(samples: PackedSamples, alphas: torch.Tensor, eps: Optional[float] = None):
    """Alpha compositing for fields that return α per interval (SDF-based
    fields): returns (weights, trans), differentiable w.r.t. α."""
    alphas = _req(alphas, torch.float32, "alphas", samples.n_samples)
    N = samples.n_samples
    rid = samples.ray_id if samples.ray_id is not None and samples.ray_id.numel() == N and N else None
    return _AlphaWeightsFn.apply(samples.packed_info, alphas, neg_log_eps(eps), rid)


class _AccumFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, packed_info, weights, values, C_, ray_id):
        n, N = packed_info.shape[0], weights.numel()
        out = torch.empty((n, C_), dtype=torch.float32, device=weights.device)
        if ray_id is not None:  # samples from the sampling calls: the flat-tile kernel
            check(L.lib().nacc_accumulate_along_rays_flat(_ptr(packed_info), _ptr(ray_id), n, _ptr(weights),
                                                          _ptr(values), C_, N, _ptr(out), _stream()),
                  "nacc_accumulate_along_rays_flat")
        else:
            check(L.lib().nacc_accumulate_along_rays(_ptr(packed_info), n, _ptr(weights), _ptr(values), C_, N,
                                                     _ptr(out), _stream()), "nacc_accumulate_along_rays")
        ctx.save_for_backward(packed_info, weights, values, ray_id)
        ctx.C = C_
        ctx.has_values = values is not None
        return out

    @staticmethod
    def backward(ctx, g_out):
        packed_info, weights, values, ray_id = ctx.saved_tensors
        n, N = packed_info.shape[0], weights.numel()
        g_w = torch.empty_like(weights)
        g_v = torch.empty_like(values) if ctx.has_values else None
        g_out = g_out.contiguous().float()
        if ray_id is not None:  # one thread per sample
            check(L.lib().nacc_accumulate_along_rays_bwd_flat(_ptr(ray_id), n, _ptr(weights),
                                                              _ptr(values if ctx.has_values else None), ctx.C, N,
                                                              _ptr(g_out), _ptr(g_w), _ptr(g_v), _stream()),
                  "nacc_accumulate_along_rays_bwd_flat")
        else:
            check(L.lib().nacc_accumulate_along_rays_bwd(_ptr(packed_info), n, _ptr(weights),
                                                         _ptr(values if ctx.has_values else None), ctx.C, N,
                                                         _ptr(g_out), _ptr(g_w), _ptr(g_v), _stream()),
                  "nacc_accumulate_along_rays_bwd")
        return None, g_w, g_v, None, None


def accumulate_along_rays(samples: PackedSamples, weights: torch.Tensor, values: Optional[torch.Tensor] = None):
    """Segmented sums out[r] = Σ_i w_i v_i (values None = ones, i.e. opacity).  Samples carrying
    ray_id (the sampling calls' output: contiguous packing) take the flat-tile kernels; an empty
    ray_id takes the one-warp-per-ray kernels (any packing)."""
    N = samples.n_samples
    weights = _req(weights, torch.float32, "weights", N)
    rid = samples.ray_id if samples.ray_id is not None and samples.ray_id.numel() == N and N else None
    if values is None:
        return _AccumFn.apply(samples.packed_info, weights, None, 1, rid)
    values = _req(values, torch.float32, "values")
    C_ = values.numel() // max(N, 1) if N else (values.shape[-1] if values.dim() > 1 else 1)
    return _AccumFn.apply(samples.packed_info, weights, values.view(N, C_) if N else values, C_, rid)


# ----------------------------------------------------------------------------- proposal resampling
MAP_IDENTITY, MAP_LINDISP = 0, 1


def importance_sample(s_edges: torch.Tensor, n_out: int, sigma: Optional[torch.Tensor] = None,
                      cdf: Optional[torch.Tensor] = None, map_kind: int = MAP_LINDISP, t_near=0.2,
                      t_far=1000.0, stratified: bool = False, seed: int = 0):
    """Inverse-CDF resampling of interval edges (Eq. 1 + Eq. 3; s-space
    P:257).  s_edges [n, m+1]; returns (s_out, t_out) [n, n_out+1].  t_near /
    t_far are scalars, or per-ray f32 tensors [n] (the combined estimator's
    spans from ``occgrid_ray_bounds``; rays with t_far <= t_near are culled)."""
    n, m1 = s_edges.shape
    s_edges = _req(s_edges, torch.float32, "s_edges")
    if sigma is not None:
        sigma = _req(sigma.detach(), torch.float32, "sigma", n * (m1 - 1))
    if cdf is not None:
        cdf = _req(cdf.detach(), torch.float32, "cdf", n * m1)
    s_out = torch.empty((n, n_out + 1), dtype=torch.float32, device=s_edges.device)
    t_out = torch.empty_like(s_out)
    if isinstance(t_near, torch.Tensor) or isinstance(t_far, torch.Tensor):
        tn = _req(t_near.detach(), torch.float32, "t_near", n)
        tf = _req(t_far.detach(), torch.float32, "t_far", n)
        check(L.lib().nacc_importance_sample_ranged(n, m1 - 1, _ptr(s_edges), _ptr(sigma), _ptr(cdf), int(map_kind),
                                                    _ptr(tn), _ptr(tf), int(n_out), int(bool(stratified)), int(seed),
                                                    _ptr(s_out), _ptr(t_out), _stream()),
              "nacc_importance_sample_ranged")
        return s_out, t_out
    check(L.lib().nacc_importance_sample(n, m1 - 1, _ptr(s_edges), _ptr(sigma), _ptr(cdf), int(map_kind),
                                         float(t_near), float(t_far), int(n_out), int(bool(stratified)), int(seed),
                                         _ptr(s_out), _ptr(t_out), _stream()), "nacc_importance_sample")
    return s_out, t_out


class _PdfLossFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t, w, th, wh, eps):
        n, nf1 = t.shape
        np1 = th.shape[1]
        loss = torch.empty(n, dtype=torch.float32, device=t.device)
        check(L.lib().nacc_pdf_loss(n, nf1 - 1, _ptr(t), _ptr(w), np1 - 1, _ptr(th), _ptr(wh), float(eps), _ptr(loss),
                                    _stream()), "nacc_pdf_loss")
        ctx.save_for_backward(t, w, th, wh)
        ctx.eps = eps
        return loss

    @staticmethod
    def backward(ctx, g_loss):
        t, w, th, wh = ctx.saved_tensors
        n, nf1 = t.shape
        np1 = th.shape[1]
        g = torch.empty_like(wh)
        g_loss = g_loss.contiguous().float()
        check(L.lib().nacc_pdf_loss_bwd(n, nf1 - 1, _ptr(t), _ptr(w), np1 - 1, _ptr(th), _ptr(wh), float(ctx.eps),
                                        _ptr(g_loss), _ptr(g), _stream()), "nacc_pdf_loss_bwd")
        return None, None, None, g, None


def pdf_loss(t: torch.Tensor, w: torch.Tensor, t_prop: torch.Tensor, w_prop: torch.Tensor, eps: float = 1e-7):
    """Proposal supervision (PDF-matching / histogram-bound loss, reading #21):
    per-ray loss [n]; differentiable w.r.t. the proposal weights only."""
    n = t.shape[0]
    t = _req(t.detach(), torch.float32, "t")
    w = _req(w.detach(), torch.float32, "w", n * (t.shape[1] - 1))
    th = _req(t_prop.detach(), torch.float32, "t_prop")
    wh = _req(w_prop, torch.float32, "w_prop", n * (th.shape[1] - 1))
    return _PdfLossFn.apply(t, w.view(n, -1), th, wh.view(n, -1), float(eps))


def occgrid_ray_bounds(rays_o: torch.Tensor, rays_d: torch.Tensor, grid: GridSpec, bits: torch.Tensor,
                       params: MarchParams, t_min: Optional[torch.Tensor] = None,
                       t_max: Optional[torch.Tensor] = None):
    """Combined estimator, grid stage (reading #18): per-ray span
    (t_near, t_far) of the intervals ``sampling_occgrid`` would emit, (0, 0)
    for culled rays, and the device count of live rays."""
    lib = L.lib()
    n = rays_o.shape[0]
    dev = rays_o.device
    rays_o = _req(rays_o, torch.float32, "rays_o", 3 * n)
    rays_d = _req(rays_d, torch.float32, "rays_d", 3 * n)
    bits = _req(bits, torch.int32, "bits")
    if t_min is not None:
        t_min = _req(t_min, torch.float32, "t_min", n)
    if t_max is not None:
        t_max = _req(t_max, torch.float32, "t_max", n)
    g, p = grid.c(), params.c()
    ws = _ws(lib.nacc_sampling_occgrid_workspace_bytes(C.byref(g), C.byref(p), n), dev)
    tn = torch.empty(n, dtype=torch.float32, device=dev)
    tf = torch.empty(n, dtype=torch.float32, device=dev)
    alive = torch.empty(1, dtype=torch.int64, device=dev)
    check(lib.nacc_occgrid_ray_bounds(C.byref(g), _ptr(bits), C.byref(p), _ptr(rays_o), _ptr(rays_d), _ptr(t_min),
                                      _ptr(t_max), n, _ptr(tn), _ptr(tf), _ptr(alive), _ptr(ws), ws.numel(),
                                      _stream()), "nacc_occgrid_ray_bounds")
    return tn, tf, alive


# ----------------------------------------------------------------------------- occupancy grid
def owner_slab(n_cells: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous owner slab of cells for `rank` (reading #25)."""
    return n_cells * rank // world, n_cells * (rank + 1) // world


def merge_fresh(slab_values: torch.Tensor, lo: int, hi: int, n_cells: int, group=None) -> torch.Tensor:
    """Owner-computes merge of the fresh grid values (reading #15):
    each rank fills its slab [lo, hi) of a zero buffer and a MAX all-reduce
    over the process group (NCCL over NVLink on GPUs) assembles the full grid.
    σ >= 0, so non-owners' zeros never win; the result is identical on every
    rank and equal to a one-rank evaluation."""
    fresh = torch.zeros(n_cells, dtype=torch.float32, device=slab_values.device)
    fresh[lo:hi] = slab_values.reshape(-1).float()
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        if torch.distributed.get_world_size(group) > 1:
            torch.distributed.all_reduce(fresh, op=torch.distributed.ReduceOp.MAX, group=group)
    return fresh


class OccupancyGrid:
    """The occupancy-grid transmittance estimator (P:240-241, P:26 ``nerfacc.
    TransmittanceEstimator``): fp32 cached density + public bitfield, updated
    with EMA (or max-decay) every n steps."""

    def __init__(self, spec: GridSpec, device="cuda", decay: float = 0.95, threshold: float = 0.01,
                 rule: int = 0, thresh_rule: int = 0, seed: int = 0):
        self.spec = spec
        self.device = torch.device(device)
        self.density = torch.zeros(spec.n_cells, dtype=torch.float32, device=self.device)
        nb = L.lib().nacc_grid_bits_bytes(C.byref(spec.c()))
        self.bits = torch.zeros(nb // 4, dtype=torch.int32, device=self.device)
        check(L.lib().nacc_grid_prepare(C.byref(spec.c()), _ptr(self.bits), _stream()), "nacc_grid_prepare")
        self.decay, self.threshold, self.rule, self.thresh_rule, self.seed = decay, threshold, rule, thresh_rule, seed
        self.mean = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._ws = _ws(L.lib().nacc_occgrid_workspace_bytes(C.byref(spec.c())), self.device)

    def points(self, step: int, jitter: bool = True, cell_begin: int = 0, cell_count: Optional[int] = None):
        if cell_count is None:
            cell_count = self.spec.n_cells - cell_begin
        xyz = torch.empty((cell_count, 3), dtype=torch.float32, device=self.device)
        g = self.spec.c()
        check(L.lib().nacc_occgrid_points(C.byref(g), self.seed, int(step), int(bool(jitter)), int(cell_begin),
                                          int(cell_count), _ptr(xyz), _stream()), "nacc_occgrid_points")
        return xyz

    def times(self, step: int, draw: int, cell_begin: int = 0, cell_count: Optional[int] = None):
        """Per-cell timestamps in [0, 1) of draw `draw` (dynamic scenes; reading #20)."""
        if cell_count is None:
            cell_count = self.spec.n_cells - cell_begin
        t = torch.empty(cell_count, dtype=torch.float32, device=self.device)
        g = self.spec.c()
        check(L.lib().nacc_occgrid_times(C.byref(g), self.seed, int(step), int(draw), int(cell_begin),
                                         int(cell_count), _ptr(t), _stream()), "nacc_occgrid_times")
        return t

    def update(self, fresh: torch.Tensor):
        fresh = _req(fresh, torch.float32, "fresh", self.spec.n_cells)
        g = self.spec.c()
        check(L.lib().nacc_occgrid_update(C.byref(g), _ptr(self.density), _ptr(fresh), int(self.rule),
                                          float(self.decay), float(self.threshold), int(self.thresh_rule),
                                          _ptr(self.bits), _ptr(self.mean), _ptr(self._ws), self._ws.numel(),
                                          _stream()), "nacc_occgrid_update")

    def update_every_n_steps(self, step: int, occ_eval_fn: Callable[..., torch.Tensor], n: int = 16,
                             jitter: bool = True, process_group=None, time_draws: int = 0) -> bool:
        """Alg. 1 ``estimator.update_every_n_steps``: every n steps,
        owner-computes the fresh values σ(x)·Δt on this rank's cell slab,
        merges them with a MAX all-reduce over the process group (the path's
        one collective; non-owners contribute 0 since σ >= 0) and applies
        the identical update on every rank.  With time_draws = K > 0 the
        scene is dynamic: occ_eval_fn(x, t) is evaluated at K
        per-cell timestamps and the draws are merged with MAX, so the grid
        holds the maximum opacity over time."""
        if step % n != 0:
            return False
        world, rank = 1, 0
        if process_group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            world = torch.distributed.get_world_size(process_group)
            rank = torch.distributed.get_rank(process_group)
        C_ = self.spec.n_cells
        lo, hi = owner_slab(C_, rank, world)
        if hi <= lo:
            vals = torch.zeros(0, dtype=torch.float32, device=self.device)
        elif time_draws <= 0:
            vals = occ_eval_fn(self.points(step, jitter, lo, hi - lo))
        else:
            x = self.points(step, jitter, lo, hi - lo)
            vals = None
            for j in range(int(time_draws)):
                v = _req(occ_eval_fn(x, self.times(step, j, lo, hi - lo)), torch.float32, "occ", hi - lo)
                if vals is None:
                    vals = v.clone()
                else:
                    max_merge(vals, v)
        self.update(merge_fresh(vals, lo, hi, C_, process_group))
        return True

    def state_dict(self):
        return {"density": self.density.clone(), "spec": dataclasses.asdict(self.spec), "decay": self.decay,
                "threshold": self.threshold, "rule": self.rule, "thresh_rule": self.thresh_rule, "seed": self.seed}


def max_merge(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """dst = max(dst, src) in place (nacc_max_merge)."""
    n = dst.numel()
    if not (dst.is_contiguous() and dst.dtype == torch.float32):
        raise ValueError("dst must be a contiguous float32 tensor")
    src = _req(src, torch.float32, "src", n)
    check(L.lib().nacc_max_merge(_ptr(dst), _ptr(src), n, _stream()), "nacc_max_merge")
    return dst


def launch_count() -> int:
    return int(L.lib().nacc_launch_count())
