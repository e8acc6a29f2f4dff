"""SURVEY §8(d).6 CPU baseline: the oracle as it stands (never tuned), timed per stage on this
host, CFG1-CFG4 at full size, on one thread and on all host cores, with the CPU model recorded.
Context only -- parity and the roofline fraction judge the GPU path.

    python tools/cpu_baseline.py [--out profiles/r2/cpu_baseline.json]

Inputs: the workloads' seeded rays and grids; CFG2 marches the bench's estimator (16 EMA updates
of the CFG2 field at the oracle's jittered cell points, bench.ema_grid_cpu); the caller's field
values come from the numpy lattice (untimed).  Stage times: march (count + fill), filter, render
fwd, render bwd; CFG4: the two resampling rounds and the 48-sample render.  All cores: median of
3 runs; one thread: one run."""
import argparse
import json
import math
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

L = -math.log(float(np.float32(1e-4)))


def timed(fn):
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


def march_pipeline(occ, levels, res, roi, o, d, field, **mkw):
    """stage-timed march -> filter -> render fwd -> render bwd (field values untimed)"""
    st = {}
    st["march"], (pk, t0, t1, rid) = timed(lambda: O.march(occ, levels, res, roi, o, d, **mkw))
    sig, _ = W.field_at_intervals(field, o, d, t0, t1, rid)
    st["filter"], (pk2, a0, a1, r2, _) = timed(lambda: O.filter_early_stop(pk, t0, t1, sig, L))
    s2, rgb = W.field_at_intervals(field, o, d, a0, a1, r2)
    st["render_fwd"], out = timed(lambda: O.render_fwd(pk2, a0, a1, s2, rgb, neg_log_eps=L))
    g = np.random.default_rng(0).normal(size=(len(pk2), 3)) * 1e-3
    st["render_bwd"], _ = timed(lambda: O.render_bwd(pk2, a0, a1, s2, rgb, g, None, None, neg_log_eps=L))
    return st, {"rays": len(o), "samples_marched": len(t0), "samples_kept": len(a0)}


def proposal_pipeline(c):
    st = {}
    n = len(c.rays_o)

    def field_dense(s_edges):
        t = W.lindisp(s_edges.astype(np.float64), c.t_near, c.t_far)
        m = 0.5 * (t[:, :-1] + t[:, 1:])
        x = c.rays_o[:, None, :].astype(np.float64) + m[..., None] * c.rays_d[:, None, :].astype(np.float64)
        sig, _ = c.scene.sigma_rgb(x.reshape(-1, 3))  # the lattice applies the contraction itself
        return sig.reshape(n, -1).astype(np.float32)

    sig1 = field_dense(c.s_edges)
    st["resample_256_96"], (s1, _) = timed(lambda: O.importance_sample(c.s_edges, 96, sigma=sig1, map_kind=1,
                                                                       t_near=c.t_near, t_far=c.t_far, want_t=False))
    s1 = s1.astype(np.float32)
    sig2 = field_dense(s1)
    st["resample_96_48"], (s2, t2) = timed(lambda: O.importance_sample(s1, 48, sigma=sig2, map_kind=1,
                                                                       t_near=c.t_near, t_far=c.t_far))
    t2 = t2.astype(np.float32)
    t0, t1 = t2[:, :-1].reshape(-1), t2[:, 1:].reshape(-1)
    pk = np.stack([np.arange(n, dtype=np.int64) * 48, np.full(n, 48, np.int64)], 1)
    rid = np.repeat(np.arange(n, dtype=np.int32), 48)
    sig, rgb = W.field_at_intervals(c.scene.sigma_rgb, c.rays_o, c.rays_d, t0, t1, rid)
    st["render_fwd"], out = timed(lambda: O.render_fwd(pk, t0, t1, sig, rgb, neg_log_eps=L))
    g = np.random.default_rng(0).normal(size=(n, 3)) * 1e-3
    st["render_bwd"], _ = timed(lambda: O.render_bwd(pk, t0, t1, sig, rgb, g, None, None, neg_log_eps=L))
    return st, {"rays": n, "samples_rendered": n * 48}


def configs():
    import bench

    c1 = W.cfg1()
    yield "cfg1", lambda: march_pipeline(c1.occ, 1, c1.res, c1.roi, c1.rays_o, c1.rays_d,
                                         lambda x: W.sphere_sigma_rgb(x), step=c1.step)
    lat, occ, step = bench.ema_grid_cpu()
    o2, d2 = W.cfg2_rays(1 << 18)
    yield "cfg2", lambda: march_pipeline(occ, 1, 128, (0, 0, 0, 1, 1, 1), o2, d2, lat.sigma_rgb, step=step)
    c3 = W.cfg3()
    field3 = c3.scene.sigma_rgb  # contracted lattice (reading #6)
    yield "cfg3", lambda: march_pipeline(c3.occ, c3.levels, c3.res, c3.roi, c3.rays_o, c3.rays_d, field3,
                                         step=c3.step, near=c3.near, cone_angle=c3.cone_angle, max_step=c3.max_step)
    c4 = W.cfg4()
    yield "cfg4", lambda: proposal_pipeline(c4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "cpu_baseline.json"))
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    res = {"kind": "oracle", "cpu_model": model, "cores": cores, "machine": platform.node(),
           "protocol": "SURVEY 8(d).6: oracle as it stands, full-size CFG1-CFG4, per stage; all cores = median "
                       "of 3 runs, one thread = one run; field values precomputed (untimed)", "configs": {}}
    for name, run in configs():
        if args.only and name != args.only:
            continue
        O.set_num_threads(cores)
        runs = []
        info = None
        for _ in range(3):
            st, info = run()
            runs.append(st)
        allc = {k: float(np.median([r[k] for r in runs])) for k in runs[0]}
        O.set_num_threads(1)
        one, _ = run()
        O.set_num_threads(cores)
        unit_n = info.get("samples_kept", info.get("samples_rendered"))
        res["configs"][name] = {**info, "stage_s_all_cores": allc, "stage_s_one_thread": one,
                                "samples_per_s_all_cores": unit_n / sum(allc.values()),
                                "samples_per_s_one_thread": unit_n / sum(one.values())}
        print(name, json.dumps(res["configs"][name]), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
