"""Run nacc_sampling_occgrid a few times on CFG2 or CFG3 (for an ncu capture of the march)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N

c = W.cfg3() if sys.argv[1:] == ["cfg3"] else W.cfg2()
spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).cuda())
o, d = torch.from_numpy(c.rays_o).cuda(), torch.from_numpy(c.rays_d).cuda()
kw = dict(step=c.step, near_plane=c.near)
if c.cone_angle:
    kw.update(cone_angle=c.cone_angle, max_step=c.max_step)
prm = N.MarchParams(**kw)
n = N.sampling_occgrid(o, d, spec, bits, prm).n_samples
for _ in range(3):
    N.sampling_occgrid(o, d, spec, bits, prm, capacity=int(n * 1.1) + 1024, sync=False)
torch.cuda.synchronize()
print("samples", n)
