"""Bench/test harness bindings (include/nacc_harness.h): the synthetic stand-in
for the user's NeRF (Alg. 1 density_fn / rgb_density_fn) and the MSE
gradient of Alg. 1 line 48.  Not part of the product path."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .api import _ptr, _req, _stream


class LatticeField:
    """Dense cell-centre lattice (σ, r, g, b) over [lo, hi]^3, trilinear
    (S:121-126), optionally queried through the scene contraction."""

    def __init__(self, data: torch.Tensor, lo: float, hi: float, contracted: bool = False):
        self.data = _req(data.float(), torch.float32, "lattice")
        self.res = int(round((self.data.numel() // 4) ** (1.0 / 3.0)))
        assert self.res ** 3 * 4 == self.data.numel()
        self.lo, self.hi, self.contracted = float(lo), float(hi), int(bool(contracted))
        self.sigma_only = self.data.view(-1, 4)[:, 0].contiguous()  # density-only lattice (4 B per cell)

    def at_samples(self, rays_o, rays_d, t0, t1, ray_id, want_rgb=True, n_dev=None):
        """σ (and rgb) at the interval midpoints; with n_dev (device int64) only
        the first *n_dev of the capacity-sized arrays are evaluated."""
        n = t0.numel()
        sigma = torch.empty(n, dtype=torch.float32, device=t0.device)
        if not want_rgb:
            st = L.harness().naccx_sigma_at_samples(_ptr(self.sigma_only), self.res, self.lo, self.hi,
                                                    self.contracted, _ptr(rays_o), _ptr(rays_d), _ptr(t0), _ptr(t1),
                                                    _ptr(ray_id), n, _ptr(n_dev), _ptr(sigma), _stream())
            if st != 0:
                raise L.NaccError(st, "naccx_sigma_at_samples")
            return sigma, None
        rgb = torch.empty((n, 3), dtype=torch.float32, device=t0.device)
        st = L.harness().naccx_field_at_samples(_ptr(self.data), self.res, self.lo, self.hi, self.contracted,
                                                _ptr(rays_o), _ptr(rays_d), _ptr(t0), _ptr(t1), _ptr(ray_id), n,
                                                _ptr(n_dev), _ptr(sigma), _ptr(rgb), _stream())
        if st != 0:
            raise L.NaccError(st, "naccx_field_at_samples")
        return sigma, rgb

    def at_points(self, xyz, scale=1.0):
        n = xyz.shape[0]
        out = torch.empty(n, dtype=torch.float32, device=xyz.device)
        st = L.harness().naccx_field_at_points(_ptr(self.data), self.res, self.lo, self.hi, self.contracted,
                                               _ptr(xyz), n, float(scale), _ptr(out), _stream())
        if st != 0:
            raise L.NaccError(st, "naccx_field_at_points")
        return out


class TextureField(LatticeField):
    """LatticeField sampled by the texture unit (hardware trilinear filtering)."""

    def __init__(self, data: torch.Tensor, lo: float, hi: float, contracted: bool = False):
        super().__init__(data, lo, hi, contracted)
        h = C.c_uint64()
        st = L.harness().naccx_tex_create(_ptr(self.data), self.res, C.byref(h), _stream())
        if st != 0:
            raise L.NaccError(st, "naccx_tex_create")
        self.handle = h.value

    def at_samples(self, rays_o, rays_d, t0, t1, ray_id, want_rgb=True, n_dev=None):
        if want_rgb:  # the float4 lattice gather measured faster than the float4 texture fetch
            return super().at_samples(rays_o, rays_d, t0, t1, ray_id, want_rgb=True, n_dev=n_dev)
        n = t0.numel()
        sigma = torch.empty(n, dtype=torch.float32, device=t0.device)
        rgb = None
        st = L.harness().naccx_tex_at_samples(self.handle, self.lo, self.hi, self.contracted, _ptr(rays_o),
                                              _ptr(rays_d), _ptr(t0), _ptr(t1), _ptr(ray_id), n, _ptr(n_dev),
                                              _ptr(sigma), _ptr(rgb), _stream())
        if st != 0:
            raise L.NaccError(st, "naccx_tex_at_samples")
        return sigma, rgb

    def __del__(self):
        try:
            L.harness().naccx_tex_destroy(self.handle)
        except Exception:
            pass


def mse_grad(color: torch.Tensor, gt: torch.Tensor) -> torch.Tensor:
    n = color.shape[0]
    g = torch.empty_like(color)
    st = L.harness().naccx_mse_grad(_ptr(color), _ptr(gt), n, _ptr(g), _stream())
    if st != 0:
        raise L.NaccError(st, "naccx_mse_grad")
    return g


def launch_count() -> int:
    return int(L.harness().naccx_launch_count())
