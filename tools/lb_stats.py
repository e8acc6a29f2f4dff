"""Look-back statistics of the CFG2 march (needs a -DNACC_LB_STATS=1 build)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N
from paper_2305_04966_b200 import _lib as L

c = W.cfg2()
spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).cuda())
o, d = torch.from_numpy(c.rays_o).cuda(), torch.from_numpy(c.rays_d).cuda()
prm = N.MarchParams(step=c.step)
f = L.lib().nacc_debug_lb_stats
out = (C.c_ulonglong * 4)()
for _ in range(3):
    N.sampling_occgrid(o, d, spec, bits, prm)
f(out)
for _ in range(5):
    N.sampling_occgrid(o, d, spec, bits, prm)
f(out)
r, polls, slept, walked = list(out)
print(f"resolves {r} polls/resolve {polls / r:.2f} sleeping polls/resolve {slept / r:.2f} tiles walked/resolve {walked / r:.1f}")
