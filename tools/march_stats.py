"""Segment-class statistics of the CFG2 / CFG3 march (needs a -DNACC_MARCH_STATS=1 build)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N
from paper_2305_04966_b200 import _lib as L

for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    c = W.cfg3() if name == "cfg3" else W.cfg2()
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).cuda())
    o, d = torch.from_numpy(c.rays_o).cuda(), torch.from_numpy(c.rays_d).cuda()
    kw = dict(step=c.step, near_plane=c.near)
    if c.cone_angle:
        kw.update(cone_angle=c.cone_angle, max_step=c.max_step)
    prm = N.MarchParams(**kw)
    f = L.lib().nacc_debug_march_stats
    out = (C.c_ulonglong * 18)()
    n = N.sampling_occgrid(o, d, spec, bits, prm).n_samples
    f(out)
    N.sampling_occgrid(o, d, spec, bits, prm, capacity=int(n * 1.1) + 1024, sync=False)
    f(out)
    v = list(out)
    nr = len(c.rays_o)
    names = ["owner slots", "skipped", "solid", "eval interior", "eval full", "eval passes", "writer passes", "tiles",
             "phase-1 passes", "emitted by eval",
             "end outside", "two-level", "level gap", "meets finer", "span > win", "non-interior", "eval->full",
             "eval->empty"]
    print(name, "rays", nr, "samples", n)
    for k, x in zip(names, v):
        print(f"  {k:16s} {x:12d}  per ray {x / nr:8.3f}")
