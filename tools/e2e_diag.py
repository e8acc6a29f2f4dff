"""Diagnose the e2e gap: raw pinned H2D / D2H bandwidth and per-step host time of the bench's e2e loop."""
import time

import torch

n = 1 << 18
h_in = torch.empty(n * 6, dtype=torch.float32).pin_memory()
d_in = torch.empty(n * 6, dtype=torch.float32, device="cuda")
h_out = torch.empty(n * 5, dtype=torch.float32).pin_memory()
d_out = torch.empty(n * 5, dtype=torch.float32, device="cuda")
for name, fn in (("h2d", lambda: d_in.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_out, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    nb = (h_in if name == "h2d" else h_out).numel() * 4
    print(f"{name}: {nb / 1e6:.1f} MB in {ms * 1e3:.1f} us = {nb / ms / 1e6:.1f} GB/s")

# ---- timeline of the bench's pipelined e2e loop (events on every stream, relative µs)
import sys

sys.path.insert(0, ".")
import bench as B

pipe = B.Pipeline(0, 1, torch.device("cuda"))
for _ in range(3):
    pipe.step()
pipe.capture()
for _ in range(3):
    pipe.step_graph()
torch.cuda.synchronize()
pinned = [(torch.from_numpy(o).pin_memory(), torch.from_numpy(d).pin_memory()) for o, d in pipe.rays_host]
main = torch.cuda.current_stream()
up, down = torch.cuda.Stream(), torch.cuda.Stream()
stage = [(torch.empty_like(pipe.o_buf), torch.empty_like(pipe.d_buf)) for _ in range(2)]
snaps = [torch.empty((n, 5), dtype=torch.float32, device="cuda") for _ in range(2)]
hosts = [torch.empty((n, 5)).pin_memory() for _ in range(2)]
E = lambda: torch.cuda.Event(enable_timing=True)
marks = []
t_host = []
z = E()
z.record()
up.wait_stream(main)
down.wait_stream(main)
h2d_done = [E() for _ in range(2)]
for i in range(8):
    b = i % 2
    h0 = time.perf_counter()
    with torch.cuda.stream(up):
        a0 = E(); a0.record(up)
        ho, hd = pinned[i % len(pinned)]
        stage[b][0].copy_(ho, non_blocking=True)
        stage[b][1].copy_(hd, non_blocking=True)
        a1 = E(); a1.record(up)
    main.wait_event(a1)
    g0 = E(); g0.record(main)
    pipe.o_buf.copy_(stage[b][0], non_blocking=True)
    pipe.d_buf.copy_(stage[b][1], non_blocking=True)
    pipe.step_graph(copy_inputs=False)
    torch.cat([pipe.outs["color"], pipe.outs["opacity"][:, None], pipe.outs["depth"][:, None]], 1, out=snaps[b])
    g1 = E(); g1.record(main)
    with torch.cuda.stream(down):
        down.wait_event(g1)
        c0 = E(); c0.record(down)
        hosts[b].copy_(snaps[b], non_blocking=True)
        c1 = E(); c1.record(down)
    t_host.append((time.perf_counter() - h0) * 1e6)
    marks.append((a0, a1, g0, g1, c0, c1))
torch.cuda.synchronize()
for i, m in enumerate(marks):
    print(f"step {i}: host {t_host[i]:7.0f} us | " + " ".join(f"{z.elapsed_time(e) * 1e3:8.0f}" for e in m))
print("columns: h2d start/end, step start/end, d2h start/end (µs since start); host = issue time")
