"""Run one §8 row a few times (for one `ncu --set full` capture of its kernels):

    python tools/prof_rows.py cfg4|grid|alpha|pdf|bounds|accum

cfg4   the proposal path: two inverse-CDF rounds 256 -> 96 -> 48 (importance_kernel) and the
       48-sample render fwd/bwd on the dense layout (render_*_warp_kernel), 2^16 rays
grid   one occupancy-grid update: points, the caller's field, EMA + threshold, mask rebuild
alpha  alpha compositing fwd/bwd over CFG2-shaped packed samples
pdf    the proposal-supervision loss fwd/bwd (2^16 rays, 48 vs 96 bins)
bounds the combined estimator's grid stage (march_bounds_kernel) on CFG2 rays
accum  granular weights fwd/bwd + accumulate_along_rays fwd/bwd on CFG2-shaped samples
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
import paper_2305_04966_b200 as N  # noqa: E402
from paper_2305_04966_b200 import harness as H  # noqa: E402

row = sys.argv[1]
dev = torch.device("cuda")
REPS = 3


def cfg2_samples(n_rays=1 << 18):
    c = W.cfg2(n_rays=n_rays)
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).to(dev))
    o, d = torch.from_numpy(c.rays_o).to(dev), torch.from_numpy(c.rays_d).to(dev)
    fld = H.TextureField(torch.from_numpy(c.scene.data.reshape(-1, 4)).to(dev), c.scene.lo, c.scene.hi)
    s = N.sampling_occgrid(o, d, spec, bits, N.MarchParams(step=c.step))
    sg, _ = fld.at_samples(o, d, s.t0, s.t1, s.ray_id, want_rgb=False)
    f = N.filter_early_stop(s, sg, 1e-4)
    sg2, rgb = fld.at_samples(o, d, f.t0, f.t1, f.ray_id)
    return c, spec, bits, o, d, f, sg2, rgb


if row == "cfg4":
    pc = W.cfg4()
    n = len(pc.rays_o)
    lat = H.LatticeField(torch.from_numpy(pc.scene.data.reshape(-1, 4)).to(dev), pc.scene.lo, pc.scene.hi,
                         contracted=True)
    o4, d4 = torch.from_numpy(pc.rays_o).to(dev), torch.from_numpy(pc.rays_d).to(dev)
    e0 = torch.from_numpy(pc.s_edges).to(dev)

    def field_dense(s_edges):
        t = 1.0 / ((1.0 - s_edges) / pc.t_near + s_edges / pc.t_far)
        m = s_edges.shape[1] - 1
        rid = torch.arange(n, device=dev, dtype=torch.int32).repeat_interleave(m)
        sig, _ = lat.at_samples(o4, d4, t[:, :-1].contiguous().view(-1), t[:, 1:].contiguous().view(-1), rid,
                                want_rgb=False)
        return sig.view(n, m)

    sig1 = field_dense(e0)
    s1, _ = N.importance_sample(e0, 96, sigma=sig1, map_kind=N.MAP_LINDISP, t_near=pc.t_near, t_far=pc.t_far)
    sig2 = field_dense(s1)
    s2, t2 = N.importance_sample(s1, 48, sigma=sig2, map_kind=N.MAP_LINDISP, t_near=pc.t_near, t_far=pc.t_far)
    t0, t1 = t2[:, :-1].contiguous().view(-1), t2[:, 1:].contiguous().view(-1)
    rid = torch.arange(n, device=dev, dtype=torch.int32).repeat_interleave(48)
    pk = torch.stack([torch.arange(n, device=dev, dtype=torch.int64) * 48,
                      torch.full((n,), 48, device=dev, dtype=torch.int64)], 1).contiguous()
    S = N.PackedSamples(pk, t0, t1, rid)
    sg, rgb = lat.at_samples(o4, d4, t0, t1, rid)
    g = torch.randn(n, 3, device=dev)
    for _ in range(REPS):
        N.importance_sample(e0, 96, sigma=sig1, map_kind=N.MAP_LINDISP, t_near=pc.t_near, t_far=pc.t_far)
        N.importance_sample(s1, 48, sigma=sig2, map_kind=N.MAP_LINDISP, t_near=pc.t_near, t_far=pc.t_far)
        col, _, _, cx = N.render_fwd(S, sg, rgb, 1e-4)
        N.render_bwd(S, sg, rgb, cx, g, None, None, 1e-4)
elif row == "grid":
    c = W.cfg2(n_rays=16)
    spec = N.GridSpec(roi=(0, 0, 0, 1, 1, 1), res=128, levels=1)
    fld = H.TextureField(torch.from_numpy(c.scene.data.reshape(-1, 4)).to(dev), c.scene.lo, c.scene.hi)
    grid = N.OccupancyGrid(spec, device=dev, decay=0.95, threshold=0.01, seed=1234)
    for k in range(REPS + 1):
        grid.update_every_n_steps(16 * k, lambda x: fld.at_points(x, c.step), n=16)
elif row == "alpha":
    c, spec, bits, o, d, f, sg2, rgb = cfg2_samples()
    alph = (-torch.expm1(-sg2 * (f.t1 - f.t0))).contiguous().requires_grad_()
    gw = torch.randn_like(alph)
    for _ in range(REPS):
        w, _ = N.render_weights_alpha(f, alph)
        (w * gw).sum().backward()
elif row == "pdf":
    n = 1 << 16
    tf48 = torch.sort(torch.rand(n, 49, device=dev), dim=1).values.contiguous()
    w48 = torch.rand(n, 48, device=dev)
    w48 = (w48 / w48.sum(1, keepdim=True)).contiguous()
    tp96 = torch.sort(torch.rand(n, 97, device=dev), dim=1).values.contiguous()
    wp96 = (0.7 * torch.rand(n, 96, device=dev)).contiguous().requires_grad_()
    for _ in range(REPS):
        N.pdf_loss(tf48, w48, tp96, wp96).sum().backward()
elif row == "bounds":
    c = W.cfg2()
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).to(dev))
    o, d = torch.from_numpy(c.rays_o).to(dev), torch.from_numpy(c.rays_d).to(dev)
    for _ in range(REPS):
        N.occgrid_ray_bounds(o, d, spec, bits, N.MarchParams(step=c.step))
elif row == "accum":
    c, spec, bits, o, d, f, sg2, rgb = cfg2_samples()
    sgr = sg2.clone().requires_grad_()
    rgbr = rgb.clone().requires_grad_()
    for _ in range(REPS):
        w, T, a = N.render_weights(f, sgr, 1e-4)
        col = N.accumulate_along_rays(f, w, rgbr)
        col.sum().backward()
else:
    raise SystemExit(__doc__)
torch.cuda.synchronize()
print("ok", row)
