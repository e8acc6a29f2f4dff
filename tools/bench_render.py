"""Time nacc_render_fwd / nacc_render_bwd alone on CFG2 post-filter samples
(oracle march + filter, harness-free numpy field): median device µs."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O
import workloads as W
import paper_2305_04966_b200 as N

c = W.cfg2()
pk, t0, t1, rid = O.march(c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step)
sig, _ = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, -np.log(np.float32(1e-4)))
s2, rgb2 = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, a0, a1, r2)
cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
S = N.PackedSamples(cu(pk2), cu(a0), cu(a1), cu(r2))
sg, rgb = cu(s2), cu(rgb2)
g = torch.randn(len(pk2), 3, device="cuda")


def timed(fn, n=40, batches=7):
    fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(batches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / n)
    return float(np.median(res)), out


ms_f, (col, _, _, cx) = timed(lambda: N.render_fwd(S, sg, rgb, 1e-4))
ms_b, _ = timed(lambda: N.render_bwd(S, sg, rgb, cx, g, None, None, 1e-4))
print(f"samples {len(a0)} render fwd {ms_f * 1e3:.1f} us bwd {ms_b * 1e3:.1f} us")
# granular render_weights forward: flat tiles (ray_id given) vs one warp per ray (empty ray_id)
with torch.no_grad():
    S0 = N.PackedSamples(S.packed_info, S.t0, S.t1, torch.zeros(0, dtype=torch.int32, device="cuda"))
    ms_wf, _ = timed(lambda: N.render_weights(S, sg, 1e-4))
    ms_ww, _ = timed(lambda: N.render_weights(S0, sg, 1e-4))
print(f"render_weights fwd flat {ms_wf * 1e3:.1f} us, warp per ray {ms_ww * 1e3:.1f} us")
# accumulate_along_rays (rgb, C = 3) forward + backward: flat vs one warp per ray
wq = torch.rand(len(a0), device="cuda", requires_grad=True)
vq = torch.rand(len(a0), 3, device="cuda", requires_grad=True)
def acc(Sx):
    o = N.accumulate_along_rays(Sx, wq, vq)
    o.backward(torch.ones_like(o))
    return o
ms_af, _ = timed(lambda: acc(S))
ms_aw, _ = timed(lambda: acc(S0))
print(f"accumulate C=3 fwd+bwd (incl. autograd) flat {ms_af * 1e3:.1f} us, warp per ray {ms_aw * 1e3:.1f} us")
# alpha compositing forward (SDF-style α): flat vs one warp per ray
aq = torch.rand(len(a0), device="cuda") * 0.2
with torch.no_grad():
    ms_pf, _ = timed(lambda: N.render_weights_alpha(S, aq, 1e-4))
    ms_pw, _ = timed(lambda: N.render_weights_alpha(S0, aq, 1e-4))
print(f"render_weights_alpha fwd flat {ms_pf * 1e3:.1f} us, warp per ray {ms_pw * 1e3:.1f} us")
# granular render_weights forward + backward (flat vs one warp per ray)
sgq = sg.clone().requires_grad_()
def wfb(Sx):
    w, T, _ = N.render_weights(Sx, sgq, 1e-4)
    (w.sum() + T.sum()).backward()
    return w
ms_bf, _ = timed(lambda: wfb(S))
ms_bw, _ = timed(lambda: wfb(S0))
print(f"render_weights fwd+bwd (incl. autograd) flat {ms_bf * 1e3:.1f} us, warp per ray {ms_bw * 1e3:.1f} us")
# alpha compositing forward + backward (flat vs one warp per ray)
aqg = aq.clone().requires_grad_()
def afb(Sx):
    w, T = N.render_weights_alpha(Sx, aqg, 1e-4)
    (w.sum() + T.sum()).backward()
    return w
ms_qf, _ = timed(lambda: afb(S))
ms_qw, _ = timed(lambda: afb(S0))
print(f"render_weights_alpha fwd+bwd (incl. autograd) flat {ms_qf * 1e3:.1f} us, warp per ray {ms_qw * 1e3:.1f} us")
