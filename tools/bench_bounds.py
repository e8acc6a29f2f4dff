"""Time nacc_occgrid_ray_bounds (combined estimator, grid stage) on CFG2 and CFG3: device µs per
call (median of batches, CUDA events)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N
sys.path.insert(0, "tools")
from bench_march_lib import timed  # noqa: E402

for name, c in (("cfg2", W.cfg2()), ("cfg3", W.cfg3())):
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).cuda())
    o, d = torch.from_numpy(c.rays_o).cuda(), torch.from_numpy(c.rays_d).cuda()
    kw = dict(step=c.step, near_plane=c.near)
    if c.cone_angle:
        kw.update(cone_angle=c.cone_angle, max_step=c.max_step)
    prm = N.MarchParams(**kw)
    ms = timed(lambda: N.occgrid_ray_bounds(o, d, spec, bits, prm))
    print(f"{name}: rays {len(c.rays_o)} ray bounds {ms * 1e3:.1f} us")
