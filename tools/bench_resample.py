"""Time nacc_importance_sample alone on CFG4 (2^16 rays, 256 -> 96 -> 48): median device µs
of CUDA-graph replays (host overhead excluded), with the algorithmic bytes per round."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W
import paper_2305_04966_b200 as N

pc = W.cfg4()
n = len(pc.rays_o)
e0 = torch.from_numpy(pc.s_edges).cuda()
g = torch.Generator(device="cuda").manual_seed(0)
sig1 = torch.rand((n, 256), device="cuda", generator=g) * 5
s1, _ = N.importance_sample(e0, 96, sigma=sig1, map_kind=N.MAP_LINDISP, t_near=pc.t_near, t_far=pc.t_far)
sig2 = torch.rand((n, 96), device="cuda", generator=g) * 5


def graph_of(fn):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    return gr


def timed(gr, reps=50, batches=7):
    res = []
    for _ in range(batches):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / reps * 1e3)
    return float(np.median(res))


for name, fn, m, k in (
        ("256->96", lambda: N.importance_sample(e0, 96, sigma=sig1, map_kind=N.MAP_LINDISP, t_near=pc.t_near,
                                                t_far=pc.t_far), 256, 96),
        ("96->48", lambda: N.importance_sample(s1, 48, sigma=sig2, map_kind=N.MAP_LINDISP, t_near=pc.t_near,
                                               t_far=pc.t_far), 96, 48)):
    us = timed(graph_of(fn))
    byts = n * (4 * (m + 1) + 4 * m + 8 * (k + 1))
    print(f"{name}: {us:.1f} us, {byts / 1e6:.1f} MB algorithmic, {byts / us / 1e3:.0f} GB/s")
