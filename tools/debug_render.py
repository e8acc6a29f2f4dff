"""Print per-output worst errors of the fused render vs the oracle at CFG2 (post-filter)."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle as O
import workloads as W
import paper_2305_04966_b200 as N
from test_gpu_parity import gpu_render, L_EPS

c = W.cfg2()
pk, t0, t1, rid = O.march(c.occ, 1, 128, c.roi, c.rays_o, c.rays_d, step=c.step)
sig, _ = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, L_EPS)
s2, rgb2 = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, a0, a1, r2)
rng = np.random.default_rng(6)
n = len(pk2)
gC, gO, gD = rng.normal(size=(n, 3)).astype(np.float32), rng.normal(size=n).astype(np.float32), \
    rng.normal(size=n).astype(np.float32)
L = -math.log(float(np.float32(1e-4)))
got = gpu_render(N, pk2, a0, a1, s2, rgb2, gC, gO, gD, 1e-4, True)
ref = O.render_fwd(pk2, a0, a1, s2, rgb2, neg_log_eps=L)
gs, grgb = O.render_bwd(pk2, a0, a1, s2, rgb2, gC, gO, gD, neg_log_eps=L)
_, margin = O.filter_counts(pk2, a0, a1, s2, L)
ok = margin >= 1e-9 * L
print("sigma max", s2.max(), "samples", len(a0))
for name, g, r in [("color", got[0], ref["color"]), ("opacity", got[1], ref["opacity"]), ("depth", got[2], ref["depth"])]:
    err = np.abs(g - r) - 1e-4 * np.abs(r) - 1e-6
    err = err.reshape(len(err), -1).max(axis=1)
    bad = np.where((err > 0) & ok)[0]
    print(name, "bad rays", len(bad), bad[:5], "worst", err.max())
    for b in bad[:3]:
        print("   ray", b, pk2[b], g[b], r[b], "margin", margin[b])
