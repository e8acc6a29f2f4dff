"""bench.py — throughput of the NerfAcc packed-sample hot path on B200.

One step = one training step of the workload's global ray batch: for every
chunk of rays, march the occupancy grid (nacc_sampling_occgrid) -> caller's
no-grad σ query (harness lattice field) -> no-gradient early-stop filter
(nacc_filter_early_stop) -> caller's σ, rgb query -> render fwd
(nacc_render_fwd) -> MSE gradient -> render bwd (nacc_render_bwd); plus the
occupancy-grid update with its MAX all-reduce every 16 steps (points ->
field -> all_reduce -> nacc_occgrid_update).

Workloads (--workload):
  cfg5       (default) BASELINE.json configs[4]: 2^24 rays per step split
             across the N ranks (strong scaling), each rank running chunks of
             2^21 rays; at N = 1 this is S(1) = 8 sequential 2^21-ray chunks
             (SURVEY §8(e)).
  cfg5-weak  2^21 rays per GPU per step (weak scaling).
  cfg2       configs[1]: 2^18 rays per GPU per step (weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5]
                    [--impl reference]

With --gpus N > 1 and no torchrun environment, the script re-launches itself
under torch.distributed.run (one rank per GPU, NCCL).  Prints ONE JSON line
(rank 0).  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import glob
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (march+render fwd+bwd) and HBM GB/s vs 8 TB/s at 1/2/4/8 B200"
UNIT = "samples/s"
UPDATE_EVERY = 16
EPS = 1e-4
GRID_DESC = ("128^3 occupancy grid over the unit box (EMA gamma 0.95, tau 0.01 on sigma*dt, 16 warm-up updates), "
             "step sqrt(3)/1024, early stop T<1e-4, dense-lattice trilinear sigma/rgb field (CFG2 scene), fwd+bwd, "
             "grid EMA update + MAX all-reduce every 16 steps")
WORKLOADS = {
    "cfg5": dict(global_rays=1 << 24, chunk=1 << 21, scaling="strong",
                 desc="cfg5: 8xB200 ray-sharded training step, 2^24 rays per step split across the GPUs "
                      "(chunks of 2^21 rays per rank), " + GRID_DESC),
    "cfg5-weak": dict(rays_per_gpu=1 << 21, chunk=1 << 21, scaling="weak",
                      desc="cfg5-weak: 2^21 rays per GPU per step, " + GRID_DESC),
    "cfg2": dict(rays_per_gpu=1 << 18, chunk=1 << 18, scaling="weak", batches=4,
                 desc="cfg2: NeRF-Synthetic-shaped training batch, 2^18 rays per GPU per step, " + GRID_DESC),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="nacc", choices=["nacc", "reference"])
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: test runs that put several ranks on one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="few steps, no extras (for ncu)")
    ap.add_argument("--eager", action="store_true", help="time the eager (non-graph) step")
    ap.add_argument("--no-extras", action="store_true", help="skip the CFG2/CFG3/CFG4 secondary measurements")
    return ap.parse_args()


def rays_per_rank(workload, world):
    w = WORKLOADS[workload]
    if "global_rays" in w:
        if w["global_rays"] % world:
            raise SystemExit(f"bench: {workload} needs a GPU count dividing 2^24, got {world}")
        return w["global_rays"] // world
    return w["rays_per_gpu"]


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args):
    """--gpus N without a torchrun environment: re-run this script under torch.distributed.run
    (one process per GPU on this node, rendezvous on 127.0.0.1) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


NCU_KERNELS_OF_STAGE = {"march": ["march_fused"], "render_fwd": ["render_fwd_warp"], "render_bwd": ["render_bwd_warp"],
                        "filter": ["filter_cut", "filter_copy"], "field_sigma": ["tex_sigma4"],
                        "field_sigma_rgb": ["field_samples"]}


def ncu_traffic(suffix=""):
    """dram read+write bytes per launch per stage, from the newest committed `ncu --set full` capture
    (profiles/<round>/ncu_traffic_bytes.json, written by tools/make_profiles.py); suffix "_cfg5"
    selects the captures taken at the CFG5 launch shape (2^21 rays per launch)."""
    rounds = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic_bytes.json")))
    if not rounds:
        return {}
    with open(rounds[-1]) as f:
        by_kernel = json.load(f)
    return {st: sum(by_kernel[k + suffix] for k in ks) for st, ks in NCU_KERNELS_OF_STAGE.items()
            if all(k + suffix in by_kernel for k in ks)}


def ncu_warp_instructions(kernel="march_fused"):
    """warp instructions per launch of `kernel` from the newest committed ncu summary, if any"""
    rounds = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_{kernel}.txt")))
    if not rounds:
        return None
    for ln in open(rounds[-1]):
        if ln.startswith("total warp instructions"):
            return float(ln.split()[-1])
    return None


# ----------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    def __init__(self, index):
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
def make_inputs(workload, rank, world):
    """Per-rank ray batches (resident in HBM during the timed region) and the MSE targets."""
    import workloads as W

    n = rays_per_rank(workload, world)
    if workload == "cfg2":
        rays = [W.cfg2_rays(n, seed=1002 + 1000 * rank + 17 * b) for b in range(WORKLOADS["cfg2"]["batches"])]
    elif workload == "cfg5":
        rays = [W.cfg5_rays(rank, world)]
    else:  # cfg5-weak: rank r's 2^21 rays are slice r of an 8 x 2^21 global draw (then a reseeded one)
        rays = [W.cfg5_rays(rank % 8, 8, seed=1005 + 1000 * (rank // 8))]
    rng = np.random.default_rng(7 + rank)
    gt = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    return rays, W.cfg2_lattice(), gt


class Pipeline:
    """One training step of the workload through the public API (paper_2305_04966_b200): the
    rank's rays in chunks, each chunk march -> σ -> filter -> σ,rgb -> render fwd -> MSE grad ->
    render bwd."""

    def __init__(self, workload, rank, world, device):
        import torch

        import workloads as W
        import paper_2305_04966_b200 as N
        from paper_2305_04966_b200 import harness as H

        self.N, self.H, self.torch = N, H, torch
        self.workload, self.rank, self.world, self.device = workload, rank, world, device
        self.n_rank = rays_per_rank(workload, world)
        ch = min(WORKLOADS[workload]["chunk"], self.n_rank)
        self.chunks = [(c, min(c + ch, self.n_rank)) for c in range(0, self.n_rank, ch)]
        rays, lat, gt = make_inputs(workload, rank, world)
        self.rays_host = rays
        self.rays = [(torch.from_numpy(o).to(device), torch.from_numpy(d).to(device)) for o, d in rays]
        self.gt = torch.from_numpy(gt).to(device)
        self.lattice = lat
        self.field = H.TextureField(torch.from_numpy(lat.data.reshape(-1, 4)).to(device), lat.lo, lat.hi)
        self.spec = N.GridSpec(roi=(0, 0, 0, 1, 1, 1), res=128, levels=1)
        self.step_size = float(np.float32(W.SQRT3 / 1024.0))
        self.params = N.MarchParams(step=self.step_size)
        self.grid = N.OccupancyGrid(self.spec, device=device, decay=0.95, threshold=0.01, seed=1234)
        self.occ_fn = lambda x: self.field.at_points(x, self.step_size)  # v = σ·Δt
        for k in range(16):  # warm the estimator (SPEC cmd_render W = 16), untimed
            self.grid.update_every_n_steps(k * UPDATE_EVERY, self.occ_fn, n=UPDATE_EVERY)
        self.capacity = None
        self.k = 0
        self.stats = {"pre": 0, "post": 0, "rays": 0}
        self.events = []

    def step_chunk(self, o, d, gt, timing=False):
        N, H, torch = self.N, self.H, self.torch
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)] if timing else None
        rec = (lambda i: ev[i].record()) if timing else (lambda i: None)
        rec(0)
        s = N.sampling_occgrid(o, d, self.spec, self.grid.bits, self.params, capacity=self.capacity)
        self.capacity = int(s.n_samples * 1.15) + 1024
        rec(1)
        sigma, _ = self.field.at_samples(o, d, s.t0, s.t1, s.ray_id, want_rgb=False)
        rec(2)
        f = N.filter_early_stop(s, sigma, EPS)
        rec(3)
        sig2, rgb = self.field.at_samples(o, d, f.t0, f.t1, f.ray_id, want_rgb=True)
        sig2.requires_grad_(True)
        rgb.requires_grad_(True)
        rec(4)
        color, opacity, depth = N.rendering(f, sig2, rgb, eps=EPS)
        rec(5)
        g = H.mse_grad(color.detach(), gt)
        rec(6)
        color.backward(g)
        rec(7)
        self.stats["pre"] += s.n_samples
        self.stats["post"] += f.n_samples
        self.stats["rays"] += s.n_rays
        if timing:
            self.events.append(ev)
        return color, opacity, depth, f.n_samples

    def step(self, rays=None, timing=False):
        """eager step (warm-up, capacity estimate, --eager)"""
        o, d = rays if rays is not None else self.rays[self.k % len(self.rays)]
        outs, post = [], 0
        for c0, c1 in self.chunks:
            color, opacity, depth, n_post = self.step_chunk(o[c0:c1], d[c0:c1], self.gt[c0:c1], timing)
            outs.append((color, opacity, depth))
            post += n_post
        self.grid.update_every_n_steps(self.k, self.occ_fn, n=UPDATE_EVERY)
        self.k += 1
        cat = self.torch.cat
        return (cat([x[0] for x in outs]), cat([x[1] for x in outs]), cat([x[2] for x in outs]), post)

    def stage_ms(self):
        """mean per-chunk stage times x chunks per step"""
        names = ["march", "field_sigma", "filter", "field_sigma_rgb", "render_fwd", "mse_grad", "render_bwd"]
        acc = {n: 0.0 for n in names}
        for ev in self.events:
            for i, n in enumerate(names):
                acc[n] += ev[i].elapsed_time(ev[i + 1])
        k = max(len(self.events), 1)
        return {n: v / k * len(self.chunks) for n, v in acc.items()}

    # ------------------------------------------------------------------ CUDA-graph step
    def capture(self):
        """Capture the step as ONE CUDA graph over static buffers (every chunk: march -> field σ
        -> filter -> field σ,rgb -> render fwd -> MSE grad -> render bwd, + counters and the
        result snapshot), using the device-count API (no host syncs); plus per-stage graphs of
        chunk 0 for the stage breakdown.  The capacity is the max total seen over the chunks x
        1.25; an overflow is recorded in a device status checked after the timed region."""
        N, H, torch = self.N, self.H, self.torch
        torch.cuda.synchronize()
        caps = []
        for o, d in self.rays:
            for c0, c1 in self.chunks:
                caps.append(N.sampling_occgrid(o[c0:c1], d[c0:c1], self.spec, self.grid.bits, self.params).n_samples)
        cap1 = int(max(caps) * 1.25) + 4096
        if len(self.rays) == 1:  # one resident batch: the graph reads it in place
            self.o_buf, self.d_buf = self.rays[0]
        else:  # rotating batches are copied into the static input each step
            self.o_buf = self.rays[0][0].clone()
            self.d_buf = self.rays[0][1].clone()
        self.acc = torch.zeros(2, dtype=torch.int64, device=self.device)  # pre, post
        self.acc_status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.result = torch.zeros((self.n_rank, 5), dtype=torch.float32, device=self.device)  # colour, opacity, depth
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        l0 = N.launch_count() + H.launch_count()

        def stages_of(c0, c1, outs):
            o, d, gt = self.o_buf[c0:c1], self.d_buf[c0:c1], self.gt[c0:c1]

            def st_march():
                outs["s"] = N.sampling_occgrid(o, d, self.spec, self.grid.bits, self.params, capacity=cap1, sync=False)

            def st_f1():
                s = outs["s"]
                outs["sigma"], _ = self.field.at_samples(o, d, s.t0, s.t1, s.ray_id, want_rgb=False, n_dev=s.total)

            def st_filter():
                outs["f"] = N.filter_early_stop(outs["s"], outs["sigma"], EPS, sync=False)

            def st_f2():
                f = outs["f"]
                outs["sig2"], outs["rgb"] = self.field.at_samples(o, d, f.t0, f.t1, f.ray_id, n_dev=f.total)

            def st_rfwd():
                outs["color"], outs["opacity"], outs["depth"], outs["ctx"] = N.render_fwd(
                    outs["f"], outs["sig2"], outs["rgb"], EPS)

            def st_mse():
                outs["gcol"] = H.mse_grad(outs["color"], gt)

            def st_rbwd():
                outs["gs"], outs["grgb"] = N.render_bwd(outs["f"], outs["sig2"], outs["rgb"], outs["ctx"],
                                                        outs["gcol"], None, None, EPS)
                self.acc[0].add_(outs["s"].total[0])
                self.acc[1].add_(outs["f"].total[0])
                torch.maximum(self.acc_status, outs["s"].status, out=self.acc_status)
                torch.cat([outs["color"], outs["opacity"][:, None], outs["depth"][:, None]], 1,
                          out=self.result[c0:c1])

            return (st_march, st_f1, st_filter, st_f2, st_rfwd, st_mse, st_rbwd)

        self.graphs = []
        self.outs0 = {}
        with torch.cuda.stream(side):
            pool = torch.cuda.graph_pool_handle()
            for fn in stages_of(*self.chunks[0], self.outs0):
                fn()  # eager warm-up of the stage on the side stream
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, pool=pool, stream=side):
                    fn()
                self.graphs.append(g)
            # the whole step as one graph (the timed path): chunks in sequence, each chunk's
            # intermediates released before the next chunk allocates (reused within the capture)
            self.full_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.full_graph, pool=torch.cuda.graph_pool_handle(), stream=side):
                for c0, c1 in self.chunks:
                    outs = {}
                    for fn in stages_of(c0, c1, outs):
                        fn()
                    del outs
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        # launches per graph step: the counter saw chunk 0's stages 2x (eager + capture) and every
        # chunk once (full capture)
        per_chunk = (N.launch_count() + H.launch_count() - l0) // (2 + len(self.chunks))
        self.launches_per_graph_step = per_chunk * len(self.chunks)
        self.capacity = cap1
        self.acc.zero_()
        self.acc_status.zero_()

    def step_graph(self, timing=False, rays=None, copy_inputs=True):
        torch = self.torch
        if copy_inputs and len(self.rays) > 1:  # else the inputs are resident in place / filled by the caller
            o, d = rays if rays is not None else self.rays[self.k % len(self.rays)]
            self.o_buf.copy_(o, non_blocking=True)
            self.d_buf.copy_(d, non_blocking=True)
        if timing:  # stage breakdown: one graph per stage of chunk 0, events between
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
            for i, g in enumerate(self.graphs):
                ev[i].record()
                g.replay()
            ev[7].record()
            self.events.append(ev)
        else:
            self.full_graph.replay()
            self.grid.update_every_n_steps(self.k, self.occ_fn, n=UPDATE_EVERY)
            self.k += 1

    def time_grid_update(self, reps=8):
        """device time of one grid update (points -> field -> MAX all-reduce -> EMA update), the
        step that runs every 16 steps"""
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            self.grid.update_every_n_steps(0, self.occ_fn, n=UPDATE_EVERY)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps


def run_extras(device, reps=20):
    """Secondary measurements of the other §8 rows (not the headline): the
    CFG3 cascaded cone march (640k rays, 4 levels), the CFG4 proposal path
    (2^16 rays, 256 -> 96 -> 48 inverse-CDF resampling, then a 48-sample render
    fwd+bwd) and the P:86 no-gradient-filtering comparison on CFG2.  Device
    time per call with CUDA events, inputs resident."""
    import torch

    import workloads as W
    import paper_2305_04966_b200 as N
    from paper_2305_04966_b200 import harness as H

    def timed(fn, n=reps, batches=5):
        """median over batches of the mean per-call device time (one slow batch does not move it)"""
        fn()
        torch.cuda.synchronize()
        per = max(n // batches, 2)
        res = []
        for _ in range(batches):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(per):
                out = fn()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / per)
        return float(np.median(res)), out

    out = {}
    peak, _ = measured_peaks()
    # ---- CFG3: cascaded grid + cone steps
    c = W.cfg3()
    spec = N.GridSpec(roi=c.roi, res=c.res, levels=c.levels)
    bits = N.prepare_bits(spec, torch.from_numpy(W.pack_bits(c.occ).view(np.int32)).to(device))
    o, d = torch.from_numpy(c.rays_o).to(device), torch.from_numpy(c.rays_d).to(device)
    prm = N.MarchParams(step=c.step, near_plane=c.near, cone_angle=c.cone_angle, max_step=c.max_step)
    n3 = N.sampling_occgrid(o, d, spec, bits, prm).n_samples
    cap = int(n3 * 1.1) + 1024
    ms3, s3 = timed(lambda: N.sampling_occgrid(o, d, spec, bits, prm, capacity=cap, sync=False))
    byts = len(c.rays_o) * 40 + n3 * 12
    out["cfg3_march"] = {"rays": len(c.rays_o), "samples": n3, "ms": ms3, "samples_per_s": n3 / (ms3 / 1e3),
                         "GBps": byts / (ms3 / 1e3) / 1e9, "frac_of_peak": byts / (ms3 / 1e3) / 1e9 / peak}
    # ---- CFG3 full inference frame (SURVEY 8(d).2 passes): march -> field σ -> filter -> field σ,rgb
    # -> render fwd, device counts throughout (no host sync inside the frame); harness field included
    fld3 = H.TextureField(torch.from_numpy(c.scene.data.reshape(-1, 4)).to(device), c.scene.lo, c.scene.hi,
                          contracted=True)

    def frame():
        s = N.sampling_occgrid(o, d, spec, bits, prm, capacity=cap, sync=False)
        sg, _ = fld3.at_samples(o, d, s.t0, s.t1, s.ray_id, want_rgb=False, n_dev=s.total)
        f = N.filter_early_stop(s, sg, EPS, sync=False)
        sg2, rgb2 = fld3.at_samples(o, d, f.t0, f.t1, f.ray_id, n_dev=f.total)
        return N.render_fwd(f, sg2, rgb2, EPS), f

    ms_fr, (_, f3) = timed(frame, n=5)
    kept3 = int(f3.total.item())
    out["cfg3_frame"] = {"rays": len(c.rays_o), "samples_marched": n3, "samples_kept": kept3, "ms": ms_fr,
                         "frames_per_s": 1e3 / ms_fr, "rays_per_s": len(c.rays_o) / (ms_fr / 1e3),
                         "kept_samples_per_s": kept3 / (ms_fr / 1e3), "includes": "harness field (texture σ, "
                         "lattice σ,rgb over the contracted scene)"}
    del fld3
    # ---- CFG4: proposal resampling 256 -> 96 -> 48 + 48-sample render fwd/bwd
    pc = W.cfg4()
    lat = H.LatticeField(torch.from_numpy(pc.scene.data.reshape(-1, 4)).to(device), pc.scene.lo, pc.scene.hi,
                         contracted=True)
    n4 = len(pc.rays_o)
    o4, d4 = torch.from_numpy(pc.rays_o).to(device), torch.from_numpy(pc.rays_d).to(device)
    e0 = torch.from_numpy(pc.s_edges).to(device)

    def lindisp(sv):
        return 1.0 / ((1.0 - sv) / pc.t_near + sv / pc.t_far)

    def field_dense(s_edges):  # caller's proposal-field query at the interval midpoints (harness)
        t = lindisp(s_edges)
        m = s_edges.shape[1] - 1
        rid = torch.arange(n4, device=device, dtype=torch.int32).repeat_interleave(m)
        sig, _ = lat.at_samples(o4, d4, t[:, :-1].contiguous().view(-1), t[:, 1:].contiguous().view(-1), rid,
                                want_rgb=False)
        return sig.view(n4, m)

    sig1 = field_dense(e0)
    ms_a, (s1, _) = timed(lambda: N.importance_sample(e0, 96, sigma=sig1, map_kind=N.MAP_LINDISP, t_near=pc.t_near,
                                                      t_far=pc.t_far))
    sig2 = field_dense(s1)
    ms_b, (s2, t2) = timed(lambda: N.importance_sample(s1, 48, sigma=sig2, map_kind=N.MAP_LINDISP, t_near=pc.t_near,
                                                       t_far=pc.t_far))
    t0 = t2[:, :-1].contiguous().view(-1)
    t1 = t2[:, 1:].contiguous().view(-1)
    rid = torch.arange(n4, device=device, dtype=torch.int32).repeat_interleave(48)
    pk = torch.stack([torch.arange(n4, device=device, dtype=torch.int64) * 48,
                      torch.full((n4,), 48, device=device, dtype=torch.int64)], 1).contiguous()
    samples = N.PackedSamples(pk, t0, t1, rid)
    sg, rgb = lat.at_samples(o4, d4, t0, t1, rid)
    ms_f, (col, opa, dep, cx) = timed(lambda: N.render_fwd(samples, sg, rgb, EPS))
    gcol = torch.randn_like(col)
    ms_r, _ = timed(lambda: N.render_bwd(samples, sg, rgb, cx, gcol, None, None, EPS))
    b_a = n4 * (4 * 257 + 4 * 256 + 8 * 97)
    b_b = n4 * (4 * 97 + 4 * 96 + 8 * 49)
    out["cfg4_proposal"] = {"rays": n4, "resample_256_96_ms": ms_a, "resample_96_48_ms": ms_b,
                            "resample_GBps": (b_a + b_b) / ((ms_a + ms_b) / 1e3) / 1e9,
                            "render_fwd_ms": ms_f, "render_bwd_ms": ms_r,
                            "rendered_samples_per_s": n4 * 48 / ((ms_f + ms_r) / 1e3),
                            "rays_per_s": n4 / ((ms_a + ms_b + ms_f + ms_r) / 1e3)}
    # ---- P:86 no-gradient filtering on CFG2: render fwd+bwd over every marched sample versus
    # filter + render over the kept ones (library time; the harness field's share reported apart)
    N2 = 1 << 18  # CFG2 ray batch
    c2 = W.cfg2(n_rays=N2)
    spec2 = N.GridSpec(roi=c2.roi, res=c2.res, levels=c2.levels)
    bits2 = N.prepare_bits(spec2, torch.from_numpy(W.pack_bits(c2.occ).view(np.int32)).to(device))
    o2, d2 = torch.from_numpy(c2.rays_o).to(device), torch.from_numpy(c2.rays_d).to(device)
    fld = H.TextureField(torch.from_numpy(c2.scene.data.reshape(-1, 4)).to(device), c2.scene.lo, c2.scene.hi)
    s_all = N.sampling_occgrid(o2, d2, spec2, bits2, N.MarchParams(step=c2.step))
    sg_all, rgb_all = fld.at_samples(o2, d2, s_all.t0, s_all.t1, s_all.ray_id)
    g_all = torch.randn((N2, 3), device=device)

    def unfiltered():
        col, _, _, cx = N.render_fwd(s_all, sg_all, rgb_all, EPS)
        return N.render_bwd(s_all, sg_all, rgb_all, cx, g_all, None, None, EPS)

    f_kept = N.filter_early_stop(s_all, sg_all, EPS, sync=False)  # capacity-sized, device total
    sg_k, rgb_k = fld.at_samples(o2, d2, f_kept.t0, f_kept.t1, f_kept.ray_id, n_dev=f_kept.total)

    def filtered():
        f = N.filter_early_stop(s_all, sg_all, EPS, sync=False)
        col, _, _, cx = N.render_fwd(f, sg_k, rgb_k, EPS)
        return N.render_bwd(f, sg_k, rgb_k, cx, g_all, None, None, EPS)

    ms_u, _ = timed(unfiltered)
    ms_k, _ = timed(filtered)
    ms_fu, _ = timed(lambda: fld.at_samples(o2, d2, s_all.t0, s_all.t1, s_all.ray_id))
    ms_fs, _ = timed(lambda: fld.at_samples(o2, d2, s_all.t0, s_all.t1, s_all.ray_id, want_rgb=False))
    ms_fk, _ = timed(lambda: fld.at_samples(o2, d2, f_kept.t0, f_kept.t1, f_kept.ray_id, n_dev=f_kept.total))
    out["no_grad_filter_P86"] = {
        "samples_marched": s_all.n_samples, "samples_kept": int(f_kept.total.item()),
        "render_fwd_bwd_all_ms": ms_u, "filter_plus_render_fwd_bwd_kept_ms": ms_k,
        "library_speedup": ms_u / ms_k,
        "harness_field_all_sigma_rgb_ms": ms_fu, "harness_field_sigma_all_plus_sigma_rgb_kept_ms": ms_fs + ms_fk,
        "speedup_with_harness_field": (ms_u + ms_fu) / (ms_k + ms_fs + ms_fk)}
    # ---- P:120-122 combined estimator on CFG2 rays: grid spans (culling), then one proposal
    # round 64 -> 32 edges inside each span (identity map), then a 32-sample render fwd+bwd
    n2, m2 = N2, 64
    prm2 = N.MarchParams(step=c2.step)
    ms_b, (tn2, tf2, alive2) = timed(lambda: N.occgrid_ray_bounds(o2, d2, spec2, bits2, prm2))
    e64 = torch.linspace(0, 1, m2 + 1, device=device).repeat(n2, 1).contiguous()
    tm = tn2[:, None] + 0.5 * (e64[:, :-1] + e64[:, 1:]) * (tf2 - tn2)[:, None]
    rid64 = torch.arange(n2, device=device, dtype=torch.int32).repeat_interleave(m2)
    sig64, _ = fld.at_samples(o2, d2, tm.reshape(-1).contiguous(), tm.reshape(-1).contiguous(), rid64,
                              want_rgb=False)
    ms_p, (s32, t32) = timed(lambda: N.importance_sample(e64, 32, sigma=sig64.view(n2, m2), map_kind=N.MAP_IDENTITY,
                                                         t_near=tn2, t_far=tf2))
    pk32 = torch.stack([torch.arange(n2, device=device, dtype=torch.int64) * 32,
                        torch.full((n2,), 32, device=device, dtype=torch.int64)], 1).contiguous()
    rid32 = torch.arange(n2, device=device, dtype=torch.int32).repeat_interleave(32)
    samp32 = N.PackedSamples(pk32, t32[:, :-1].contiguous().view(-1), t32[:, 1:].contiguous().view(-1), rid32)
    sg32, rgb32 = fld.at_samples(o2, d2, samp32.t0, samp32.t1, rid32)
    ms_rf, (col32, _, _, cx32) = timed(lambda: N.render_fwd(samp32, sg32, rgb32, EPS))
    ms_rb, _ = timed(lambda: N.render_bwd(samp32, sg32, rgb32, cx32, g_all, None, None, EPS))
    # ---- alpha path (SDF-style fields) on the kept CFG2 samples, and the proposal-supervision
    # loss on CFG4-shaped histograms (48 final vs 96 proposal bins, 2^16 rays)
    n_kept = int(f_kept.total.item())
    pk_k = N.PackedSamples(f_kept.packed_info, f_kept.t0[:n_kept], f_kept.t1[:n_kept], f_kept.ray_id[:n_kept])
    alph = (-torch.expm1(-sg_k[:n_kept] * (pk_k.t1 - pk_k.t0))).contiguous()
    alph_g = alph.clone().requires_grad_()
    gw_a = torch.randn_like(alph)

    def alpha_fwd_bwd():
        w_a, _ = N.render_weights_alpha(pk_k, alph_g, eps=EPS)
        (w_a * gw_a).sum().backward()
        return w_a

    ms_al, _ = timed(alpha_fwd_bwd)
    tf48 = torch.sort(torch.rand(n4, 49, device=device), dim=1).values.contiguous()
    w48 = torch.rand(n4, 48, device=device)
    w48 = (w48 / w48.sum(1, keepdim=True)).contiguous()
    tp96 = torch.sort(torch.rand(n4, 97, device=device), dim=1).values.contiguous()
    wp96 = torch.rand(n4, 96, device=device)
    wp96 = (0.7 * wp96 / wp96.sum(1, keepdim=True)).contiguous().requires_grad_()

    def pdf_fwd_bwd():
        lp = N.pdf_loss(tf48, w48, tp96, wp96)
        lp.sum().backward()
        return lp

    ms_pdf, _ = timed(pdf_fwd_bwd)
    out["alpha_path"] = {"samples": n_kept, "weights_alpha_fwd_bwd_ms": ms_al,
                         "samples_per_s": n_kept / (ms_al / 1e3), "note": "includes autograd glue"}
    out["pdf_loss"] = {"rays": n4, "final_bins": 48, "proposal_bins": 96, "fwd_bwd_ms": ms_pdf,
                       "rays_per_s": n4 / (ms_pdf / 1e3), "note": "includes autograd glue"}
    n_alive = int(alive2.item())
    out["combined_estimator_P120"] = {
        "rays": n2, "rays_alive_after_grid": n_alive, "culled_fraction": 1.0 - n_alive / n2,
        "mean_span_alive": float(((tf2 - tn2)[tf2 > tn2]).mean().item()), "ray_bounds_ms": ms_b, "proposal_64_to_32_ms": ms_p,
        "render_fwd_ms": ms_rf, "render_bwd_ms": ms_rb,
        "library_ms": ms_b + ms_p + ms_rf + ms_rb,
        "rays_per_s": n2 / ((ms_b + ms_p + ms_rf + ms_rb) / 1e3)}
    return out


def algorithmic_bytes(stage, pre, post, rays):
    """SURVEY §8(d).4 / DESIGN.md §6: bytes the method must move, per launch."""
    if stage == "march":
        return rays * (24 + 16) + pre * 12
    if stage == "filter":
        return rays * 32 + post * 12 * 2 + rays * 16
    if stage == "render_fwd":
        return post * 24 + rays * (16 + 20 + 40)
    if stage == "render_bwd":
        return post * 40 + rays * (16 + 12 + 40)
    return None


# ----------------------------------------------------------------------------- oracle (CPU baseline)
def oracle_stages(inp):
    """march -> filter -> render fwd -> render bwd on the CPU oracle; per-stage seconds and the
    number of post-filter samples."""
    import oracle as O

    t = [time.perf_counter()]
    pk, t0, t1, rid = O.march(inp["occ"], 1, 128, (0, 0, 0, 1, 1, 1), inp["o"], inp["d"], step=inp["step"])
    t.append(time.perf_counter())
    pk2, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, inp["sig"], inp["L"])
    t.append(time.perf_counter())
    out = O.render_fwd(pk2, a0, a1, inp["s2"], inp["rgb"], neg_log_eps=inp["L"])
    t.append(time.perf_counter())
    g = 2.0 * (out["color"] - inp["gt"]) / (3 * len(pk2))
    O.render_bwd(pk2, a0, a1, inp["s2"], inp["rgb"], g, None, None, neg_log_eps=inp["L"])
    t.append(time.perf_counter())
    names = ("march", "filter", "render_fwd", "render_bwd")
    return {n: t[i + 1] - t[i] for i, n in enumerate(names)}, len(a0)


def oracle_inputs_from_gpu(pipe, n_rays):
    """The GPU arm's identical inputs for the oracle: the first n_rays rays of the rank's batch, the
    same (EMA-trained) occupancy grid, and the σ / rgb the same harness field returned for the
    same samples (the oracle's march is bit-exact with the GPU's, asserted)."""
    import torch

    N = pipe.N
    o, d = pipe.rays[0][0][:n_rays].contiguous(), pipe.rays[0][1][:n_rays].contiguous()
    s = N.sampling_occgrid(o, d, pipe.spec, pipe.grid.bits, pipe.params)
    sig, _ = pipe.field.at_samples(o, d, s.t0, s.t1, s.ray_id, want_rgb=False)
    f = N.filter_early_stop(s, sig, EPS)
    s2, rgb = pipe.field.at_samples(o, d, f.t0, f.t1, f.ray_id, want_rgb=True)
    bits = pipe.grid.bits[: (pipe.spec.n_cells + 31) // 32].cpu().numpy().view(np.uint8)
    occ = np.unpackbits(bits, bitorder="little")[: pipe.spec.n_cells].astype(np.uint8)
    torch.cuda.synchronize()
    return dict(o=o.cpu().numpy(), d=d.cpu().numpy(), occ=occ, step=pipe.step_size, sig=sig.cpu().numpy(),
                s2=s2.detach().cpu().numpy(), rgb=rgb.detach().cpu().numpy(), L=-math.log(float(np.float32(EPS))),
                gt=pipe.gt[:n_rays].cpu().numpy().astype(np.float64), n_pre=s.n_samples, n_post=f.n_samples)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(pipe, n_rays=1 << 15, reps=3):
    """The oracle as it stands on this host (bounded): the GPU arm's identical inputs
    (rays, EMA grid, field values), timed per stage on all host cores (median of `reps`) and on one
    thread (one rep)."""
    import oracle as O

    inp = oracle_inputs_from_gpu(pipe, n_rays)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    O.set_num_threads(cores)
    st, post = oracle_stages(inp)  # warm (also the parity check below)
    if post != inp["n_post"]:
        raise RuntimeError("oracle and GPU disagree on the CPU-baseline sample")
    runs = [oracle_stages(inp)[0] for _ in range(reps)]
    per = {k: float(np.median([r[k] for r in runs])) for k in runs[0]}
    O.set_num_threads(1)
    one = oracle_stages(inp)[0]
    O.set_num_threads(cores)
    tot, tot1 = sum(per.values()), sum(one.values())
    return {"value": post / tot, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n_rays} rays of the rank-0 batch, same EMA grid and harness field values as the GPU "
                      f"arm ({inp['n_pre']} marched / {post} kept samples); march+filter+render fwd+bwd",
            "stage_s_all_cores": per, "one_thread": {"value": post / tot1, "stage_s": one},
            "cpu_model": cpu_model()}


def ema_grid_cpu():
    """The GPU arm's estimator built on the CPU (reference arm): 16 EMA updates of the CFG2 field at
    the oracle's jittered cell points (same seed, decay, threshold and v = σ·Δt)."""
    import oracle as O
    import workloads as W

    lat = W.cfg2_lattice()
    step = float(np.float32(W.SQRT3 / 1024.0))
    dens = np.zeros(128 ** 3, np.float32)
    occ = None
    for k in range(16):
        x = O.occgrid_points(1, 128, (0, 0, 0, 1, 1, 1), 1234, k * UPDATE_EVERY, 1)
        v = (lat.sigma_rgb(x.astype(np.float64))[0] * step).astype(np.float32)
        dens, occ, _ = O.occgrid_update(1, 128, (0, 0, 0, 1, 1, 1), dens, v, decay=0.95, threshold=0.01)
    return lat, occ, step


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    import workloads as W

    lat, occ, step = ema_grid_cpu()
    L = -math.log(float(np.float32(EPS)))

    def sample(n):
        o, d = W.cfg5_rays(0, 8) if args.workload != "cfg2" else W.cfg2_rays(1 << 18)
        o, d = o[:n], d[:n]
        pk, t0, t1, rid = O.march(occ, 1, 128, (0, 0, 0, 1, 1, 1), o, d, step=step)
        sig, _ = W.field_at_intervals(lat.sigma_rgb, o, d, t0, t1, rid)
        _, a0, a1, r2, _ = O.filter_early_stop(pk, t0, t1, sig, L)
        s2, rgb = W.field_at_intervals(lat.sigma_rgb, o, d, a0, a1, r2)
        gt = np.random.default_rng(7).uniform(0, 1, (n, 3))
        return dict(o=o, d=d, occ=occ, step=step, sig=sig, s2=s2, rgb=rgb, L=L, gt=gt)

    # size each step so the whole --steps K --warmup W run stays within ~2 minutes
    probe = sample(4096)
    st, _ = oracle_stages(probe)
    per_ray = sum(st.values()) / 4096
    budget = 90.0 / max(args.steps + args.warmup, 1)
    n = int(min(1 << 16, max(256, budget / max(per_ray, 1e-9))))
    n = 1 << int(math.floor(math.log2(n)))
    inp = sample(n)
    for _ in range(args.warmup):
        oracle_stages(inp)
    t = time.perf_counter()
    post = 0
    for _ in range(args.steps):
        post += oracle_stages(inp)[1]
    dt = time.perf_counter() - t
    value = post / dt
    w = WORKLOADS[args.workload]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w["desc"], "rays_per_step": n,
                       "parallelism": "oracle on host cores (rank 0 only)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle",
                             "sample": f"{n} rays of the workload per step (EMA grid built on the CPU; "
                                       f"numpy field values precomputed, untimed)", "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- main arm
def run_nacc(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    n_dev = torch.cuda.device_count()
    if args.backend == "nccl" and local >= n_dev:
        raise SystemExit(f"bench: rank {rank} needs GPU {local}, only {n_dev} visible")
    torch.cuda.set_device(local % n_dev)
    device = torch.device("cuda", local % n_dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=device)
        else:
            dist.init_process_group("gloo", init_method="env://")
    import paper_2305_04966_b200 as N
    from paper_2305_04966_b200 import harness as H

    pipe = Pipeline(args.workload, rank, world, device)
    for _ in range(max(args.warmup, 3)):
        pipe.step()
    torch.cuda.synchronize()
    use_graph = not args.profile and not args.eager
    if use_graph:
        pipe.capture()
        for _ in range(3):
            pipe.step_graph()
        torch.cuda.synchronize()
        pipe.acc.zero_()
        pipe.acc_status.zero_()
    step = pipe.step_graph if use_graph else pipe.step

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-timed region: inputs resident in HBM
    pipe.stats = {"pre": 0, "post": 0, "rays": 0}
    pipe.events = []
    k_start = pipe.k
    l0 = N.launch_count() + H.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local % n_dev) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    launches = N.launch_count() + H.launch_count() - l0
    n_updates = sum(1 for k in range(k_start, k_start + args.steps) if k % UPDATE_EVERY == 0)
    if use_graph:
        launches += pipe.launches_per_graph_step * args.steps
        pre_s, post_s = pipe.acc.tolist()
        if int(pipe.acc_status.item()) != 0:
            raise RuntimeError("march capacity overflow inside the captured step; increase the capacity margin")
        stats = {"pre": pre_s, "post": post_s, "rays": pipe.n_rank * args.steps}
    else:
        stats = dict(pipe.stats)
    ms = e0.elapsed_time(e1)
    if use_graph:  # stage breakdown (not the headline): per-stage graphs with events between them
        for _ in range(min(args.steps, 50) if len(pipe.chunks) == 1 else 10):
            pipe.step_graph(timing=True)
        torch.cuda.synchronize()
    stages = pipe.stage_ms() if not args.profile else {}
    if stages:
        stages["grid_update_every_16"] = pipe.time_grid_update()
    t = torch.tensor([ms, stats["post"], stats["pre"], stats["rays"]], dtype=torch.float64, device=device)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        t[0] = tmax[0]
    ms_max, post_all, pre_all, rays_all = t.tolist()
    value = post_all / (ms_max / 1e3)

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.profile:
        pinned = [(torch.from_numpy(o).pin_memory(), torch.from_numpy(d).pin_memory()) for o, d in pipe.rays_host]
        nr = pipe.n_rank
        k2 = max(args.steps, 20) if len(pipe.chunks) == 1 else max(args.steps, 8)
        if use_graph:
            pipe.acc.zero_()
        barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        stage = [(torch.empty_like(pipe.o_buf), torch.empty_like(pipe.d_buf)) for _ in range(2)] if use_graph else None
        snaps = [torch.empty((nr, 5), dtype=torch.float32, device=device) for _ in range(2)]
        hosts = [torch.empty((nr, 5), dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        stage_free = [torch.cuda.Event() for _ in range(2)]
        snap_ready = [torch.cuda.Event() for _ in range(2)]
        d2h_done = [torch.cuda.Event() for _ in range(2)]

        def run_io(k2):
            n_post_eager = 0
            if use_graph:
                # Pipelined host I/O (what a training loop does): step i+1's rays go host->device on
                # one copy stream and step i's colour/opacity/depth device->host on another while
                # step i computes; every step still moves its own inputs and results.
                up.wait_stream(main)
                down.wait_stream(main)

                def h2d(i):
                    b = i % 2
                    with torch.cuda.stream(up):
                        if i >= 2:
                            up.wait_event(stage_free[b])  # step i-2 has copied this staging buffer out
                        ho, hd = pinned[i % len(pinned)]
                        stage[b][0].copy_(ho, non_blocking=True)
                        stage[b][1].copy_(hd, non_blocking=True)
                        h2d_done[b].record(up)

                h2d(0)
                for i in range(k2):
                    b = i % 2
                    if i + 1 < k2:
                        h2d(i + 1)
                    main.wait_event(h2d_done[b])
                    pipe.o_buf.copy_(stage[b][0], non_blocking=True)
                    pipe.d_buf.copy_(stage[b][1], non_blocking=True)
                    stage_free[b].record(main)
                    pipe.step_graph(copy_inputs=False)
                    if i >= 2:
                        main.wait_event(d2h_done[b])  # step i-2's result has left this snapshot
                    snaps[b].copy_(pipe.result, non_blocking=True)
                    snap_ready[b].record(main)
                    with torch.cuda.stream(down):
                        down.wait_event(snap_ready[b])
                        hosts[b].copy_(snaps[b], non_blocking=True)
                        d2h_done[b].record(down)
                main.wait_stream(up)
                main.wait_stream(down)
            else:
                for i in range(k2):
                    ho, hd = pinned[i % len(pinned)]
                    o = ho.to(device, non_blocking=True)
                    d = hd.to(device, non_blocking=True)
                    color, opacity, depth, n_post = pipe.step(rays=(o, d))
                    n_post_eager += n_post
                    res = torch.cat([color.detach(), opacity.detach()[:, None], depth.detach()[:, None]], 1)
                    hosts[0].copy_(res, non_blocking=True)
            return n_post_eager

        run_io(3)  # untimed: first use of the copy streams, staging buffers and pinned outputs
        torch.cuda.synchronize()
        if use_graph:
            pipe.acc.zero_()
        barrier()
        f0.record()
        h0 = time.perf_counter()
        post_e2e = run_io(k2)
        f1.record()
        host_ms = (time.perf_counter() - h0) * 1e3 / k2  # host time to issue one step
        torch.cuda.synchronize()
        barrier()
        if use_graph:
            post_e2e = int(pipe.acc[1].item())
        ms2 = f0.elapsed_time(f1)
        t2 = torch.tensor([ms2, post_e2e], dtype=torch.float64, device=device)
        if world > 1:
            m = t2.clone()
            dist.all_reduce(m[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t2[1:], op=dist.ReduceOp.SUM)
            t2[0] = m[0]
        e2e = {"value": t2[1].item() / (t2[0].item() / 1e3), "unit": UNIT, "h2d_bytes_per_step": nr * 24,
               "d2h_bytes_per_step": nr * 20, "steps": k2, "host_issue_ms_per_step": host_ms,
               "io": ("pinned host buffers; H2D of step i+1 and D2H of step i on two copy streams, "
                      "double-buffered, overlapping step i" if use_graph else "pinned host buffers, serial")}

    if rank == 0:
        peak, peak_kind = measured_peaks()
        K = args.steps
        n_chunks = len(pipe.chunks)
        pre_pg, post_pg, rays_pg = stats["pre"] / K, stats["post"] / K, stats["rays"] / K
        # per-launch (per-chunk) figures: the library kernels run once per chunk
        pre_pc, post_pc, rays_pc = pre_pg / n_chunks, post_pg / n_chunks, rays_pg / n_chunks
        roof, lib_ms, lib_bytes = None, None, None
        if stages:
            lib_stages = {k: v for k, v in stages.items() if algorithmic_bytes(k, 1, 1, 1) is not None}
            dom = max(lib_stages, key=lib_stages.get)
            byts = algorithmic_bytes(dom, pre_pc, post_pc, rays_pc)
            ms_launch = lib_stages[dom] / n_chunks
            achieved = byts / (ms_launch / 1e3) / 1e9
            # traffic from a capture at this launch shape when one is committed (CFG5: 2^21 rays)
            shape = "_cfg5" if rays_pc == (1 << 21) else ""
            tr = ncu_traffic(shape).get(dom) if shape else None
            note = ("ncu dram bytes of one launch at this shape (profiles/, CFG5 chunk of 2^21 rays)"
                    if tr else None)
            if tr is None:
                shape = ""
                tr = ncu_traffic().get(dom)
                note = "ncu dram bytes per launch of the committed CFG2 capture (profiles/), the same kernel at " \
                       "2^18 rays" if tr else None
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": tr, "kernel": dom, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": byts,
                    "ms_per_launch": ms_launch, "traffic_note": note}
            # the march is bound by instruction issue, not HBM (DESIGN.md §6/§10): its warp
            # instructions per launch (committed ncu capture, CFG2 shape) over the issue peak of
            # 148 SMs x 4 schedulers x 1 warp-instruction per cycle at the sampled SM clock
            winst = ncu_warp_instructions("march_fused" + shape) if dom == "march" else None
            if winst and rays_pc == (1 << (21 if shape else 18)):
                sm_mhz = clk.summary().get("sm_mhz") or 1965.0
                n_sm = torch.cuda.get_device_properties(device).multi_processor_count
                issue_peak = n_sm * 4 * sm_mhz * 1e6
                got = winst / (ms_launch / 1e3)
                roof["issue"] = {"warp_instructions_per_launch": winst, "achieved": got / 1e9,
                                 "peak": issue_peak / 1e9, "unit": "G warp-instr/s", "frac": got / issue_peak}
            # library stages only (march, filter, render fwd/bwd; harness field and grid update excluded),
            # from the per-stage breakdown (includes inter-graph gaps, so conservative)
            lib_ms = sum(lib_stages.values())
            lib_bytes = sum(algorithmic_bytes(k, pre_pg, post_pg, rays_pg) for k in lib_stages)
        cpu = None
        if not args.no_cpu_baseline and not args.profile and world == 1:
            cpu = cpu_baseline(pipe)
        extras = None
        if not args.profile and not args.no_extras:
            try:
                extras = run_extras(device)
                if args.workload != "cfg2":
                    extras["cfg2_step"] = cfg2_step_line(device)
            except Exception as exc:  # secondary lines never sink the headline
                extras = {"error": repr(exc)}
        clocks = clk.summary()
        w = WORKLOADS[args.workload]
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
                "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": w["desc"], "rays_per_gpu": pipe.n_rank, "chunks_per_gpu": n_chunks,
                           "global_rays_per_step": rays_all / K, "grid": "1x128^3",
                           "parallelism": f"dp{world} (ray-sharded, replicated grid, MAX all-reduce every 16 steps)",
                           "backend": args.backend if world > 1 else None,
                           "l2": "inputs larger than L2 (march output ~0.25 GB per 2^18 rays; "
                                 f"{pipe.n_rank} resident rays per GPU)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
                "execution": "one CUDA graph per step, device-count API (no host syncs)" if use_graph else "eager",
                "grid_updates_in_timed_region": n_updates,
                "samples_pre_filter_per_step_per_gpu": pre_pg, "samples_post_filter_per_step_per_gpu": post_pg,
                "pre_filter_samples_per_s": pre_all / (ms_max / 1e3), "rays_per_s": rays_all / (ms_max / 1e3),
                "stage_ms": stages, "extras": extras,
                "library_ms_per_step": lib_ms,
                "library_samples_per_s": post_pg / (lib_ms / 1e3) if lib_ms else None,
                "library_hbm": ({"algorithmic_bytes_per_step": lib_bytes, "GBps": lib_bytes / (lib_ms / 1e3) / 1e9,
                                 "frac_of_measured_peak": lib_bytes / (lib_ms / 1e3) / 1e9 / peak,
                                 "frac_of_8TBps": lib_bytes / (lib_ms / 1e3) / 8e12} if lib_ms else None)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cfg2_step_line(device, steps=100):
    """The CFG2 step (configs[1], 2^18 rays) as a secondary line when the headline is CFG5."""
    import torch

    p = Pipeline("cfg2", 0, 1, device)
    for _ in range(3):
        p.step()
    p.capture()
    for _ in range(3):
        p.step_graph()
    torch.cuda.synchronize()
    p.acc.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        p.step_graph()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    pre, post = p.acc.tolist()
    for _ in range(50):
        p.step_graph(timing=True)
    torch.cuda.synchronize()
    return {"rays": 1 << 18, "ms_per_step": ms, "samples_per_s": post / steps / (ms / 1e3),
            "samples_pre_filter_per_step": pre / steps, "samples_post_filter_per_step": post / steps,
            "stage_ms": p.stage_ms()}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_nacc(args)


if __name__ == "__main__":
    main()
