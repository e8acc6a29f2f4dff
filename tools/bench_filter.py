"""Time nacc_filter_early_stop alone on CFG2 march output (oracle march, numpy field):
median device µs of a CUDA-graph replay (host overhead excluded)."""
import math
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
sig = np.ascontiguousarray(sig, dtype=np.float32)
cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
S = N.PackedSamples(cu(pk), cu(t0), cu(t1), cu(rid))
sg = cu(sig)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    N.filter_early_stop(S, sg, 1e-4, sync=False)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        out = N.filter_early_stop(S, sg, 1e-4, sync=False)
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
res = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 40)
ref_pk, *_ = O.filter_early_stop(pk, t0, t1, sig, -math.log(float(np.float32(1e-4))))
assert np.array_equal(out.packed_info.cpu().numpy(), ref_pk), "filter parity"
print(f"samples {len(t0)} kept {int(out.total.item())} filter {np.median(res) * 1e3:.1f} us")
