"""World-size-2 runs of the real GPU path on one B200 (gloo process group, both ranks on cuda:0):
the library's OccupancyGrid.update_every_n_steps (owner-computes points -> field -> MAX
all-reduce -> nacc_occgrid_update, reading #25) must leave every rank with a
grid bit-identical to a one-rank run, and `bench.py --gpus 2` must launch two ranks that time
the step together."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _field(torch):
    # a caller's density field on the GPU: a Gaussian blob, σ(x)·Δt
    return lambda x: torch.exp(-4.0 * (x.double() ** 2).sum(1)).float() * 3.0


def _grid_after_updates(torch, N, dev):
    spec = N.GridSpec(roi=(-1, -1, -1, 1, 1, 1), res=32, levels=2)
    g = N.OccupancyGrid(spec, device=dev, decay=0.9, threshold=0.05, seed=21)
    for k in range(3):
        g.update_every_n_steps(16 * k, _field(torch), n=16)
    torch.cuda.synchronize()
    return g.density.cpu().numpy(), g.bits.cpu().numpy()


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2305_04966_b200 as N

    dens, bits = _grid_after_updates(torch, N, torch.device("cuda", 0))
    np.save(os.path.join(out_dir, f"dens{rank}.npy"), dens)
    np.save(os.path.join(out_dir, f"bits{rank}.npy"), bits)
    dist.barrier()
    dist.destroy_process_group()


def test_occgrid_update_world2_matches_one_rank(tmp_path):
    import torch
    import torch.multiprocessing as mp

    import __graft_entry__

    __graft_entry__.build()
    import paper_2305_04966_b200 as N

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    d1, b1 = _grid_after_updates(torch, N, torch.device("cuda", 0))
    assert (np.unpackbits(b1.view(np.uint8)).sum()) > 100
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"dens{r}.npy"), d1)
        assert np.array_equal(np.load(tmp_path / f"bits{r}.npy"), b1)


def test_bench_gpus2_launches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--workload", "cfg2", "--steps", "4", "--warmup", "3", "--no-extras", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["global_rays_per_step"] == 2 * (1 << 18)
    assert d["e2e"]["value"] > 0 and d["grid_updates_in_timed_region"] >= 0
