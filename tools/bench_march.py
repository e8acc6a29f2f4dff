"""Time nacc_sampling_occgrid alone on CFG2 (bench grid stand-in: the workloads
occupancy) and CFG3 (cascaded cone march): device ms per call, CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N


def timed(fn, n=40, batches=7):
    """median over batches of the mean per-call device time (ms)"""
    fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(batches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / n)
    return float(np.median(res))


for name, c in (("cfg2", W.cfg2()), ("cfg3", W.cfg3())):
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).cuda())
    o, d = torch.from_numpy(c.rays_o).cuda(), torch.from_numpy(c.rays_d).cuda()
    kw = dict(step=c.step, near_plane=c.near)
    if c.cone_angle:
        kw.update(cone_angle=c.cone_angle, max_step=c.max_step)
    prm = N.MarchParams(**kw)
    n = N.sampling_occgrid(o, d, spec, bits, prm).n_samples
    cap = int(n * 1.1) + 1024
    ms = timed(lambda: N.sampling_occgrid(o, d, spec, bits, prm, capacity=cap, sync=False))
    print(f"{name}: rays {len(c.rays_o)} samples {n} march {ms * 1e3:.1f} us")
