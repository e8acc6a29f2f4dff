"""Multi-process (world size 2, gloo, CPU) coverage of the path's one exchange
step: owner-computes cell slabs + MAX all-reduce.  The merged
fresh values, and therefore the grid update (done here by the oracle), are
identical on every rank and bit-identical to a one-rank run."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2305_04966_b200.api import merge_fresh, owner_slab

    levels, res, roi = 2, 16, (-1, -1, -1, 1, 1, 1)
    n = levels * res**3
    lo, hi = owner_slab(n, rank, world)
    xyz = O.occgrid_points(levels, res, roi, seed=5, step=16, jitter=1, cell_begin=lo, cell_count=hi - lo)
    sig = np.exp(-4 * np.sum(xyz.astype(np.float64) ** 2, axis=1)) * 3.0  # a Gaussian blob σ(x)·Δt
    fresh = merge_fresh(torch.from_numpy(sig.astype(np.float32)), lo, hi, n).numpy()
    dens = np.full(n, 0.02, np.float32)
    d2, bits, mean = O.occgrid_update(levels, res, roi, dens, fresh, decay=0.95, threshold=0.05)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.concatenate([fresh, d2, bits.astype(np.float32)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_owner_computes_max_merge_gloo(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    assert np.array_equal(outs[0], outs[1])
    # one-rank reference
    import oracle as O

    levels, res, roi = 2, 16, (-1, -1, -1, 1, 1, 1)
    n = levels * res**3
    xyz = O.occgrid_points(levels, res, roi, seed=5, step=16, jitter=1)
    sig = (np.exp(-4 * np.sum(xyz.astype(np.float64) ** 2, axis=1)) * 3.0).astype(np.float32)
    d2, bits, _ = O.occgrid_update(levels, res, roi, np.full(n, 0.02, np.float32), sig, decay=0.95, threshold=0.05)
    assert np.array_equal(outs[0], np.concatenate([sig, d2, bits.astype(np.float32)]))
    assert 0 < bits.mean() < 1


def test_owner_slabs_partition_cells():
    from paper_2305_04966_b200.api import owner_slab

    for n in (1, 7, 128**3, 4 * 128**3):
        for world in (1, 2, 3, 8):
            slabs = [owner_slab(n, r, world) for r in range(world)]
            assert slabs[0][0] == 0 and slabs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))


def _worker_dynamic(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2305_04966_b200.api import merge_fresh, owner_slab

    levels, res, roi, K = 1, 16, (0, 0, 0, 1, 1, 1), 5
    n = levels * res**3
    lo, hi = owner_slab(n, rank, world)
    xyz = O.occgrid_points(levels, res, roi, seed=9, step=0, jitter=1, cell_begin=lo, cell_count=hi - lo)
    slab = None
    for j in range(K):  # dynamic scene (reading #20): max over time draws, then the cross-rank MAX
        t = O.occgrid_times(levels, res, roi, 9, 0, j, cell_begin=lo, cell_count=hi - lo).astype(np.float64)
        c = np.stack([0.3 + 0.4 * t, np.full_like(t, 0.5), np.full_like(t, 0.5)], 1)
        v = np.where(np.linalg.norm(xyz - c, axis=1) < 0.2, 2.0, 0.0).astype(np.float32)
        slab = v if slab is None else np.maximum(slab, v)
    fresh = merge_fresh(torch.from_numpy(slab), lo, hi, n).numpy()
    np.save(os.path.join(out_dir, f"dyn{rank}.npy"), fresh)
    dist.barrier()
    dist.destroy_process_group()


def test_dynamic_grid_merge_gloo(tmp_path):
    """Time draws merged by MAX on each rank's slab, then the cross-rank MAX:
    identical on both ranks and equal to the one-rank max over the draws."""
    port = _free_port()
    mp.spawn(_worker_dynamic, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    a, b = np.load(tmp_path / "dyn0.npy"), np.load(tmp_path / "dyn1.npy")
    assert np.array_equal(a, b)
    import oracle as O

    xyz = O.occgrid_points(1, 16, (0, 0, 0, 1, 1, 1), seed=9, step=0, jitter=1)
    ref = None
    for j in range(5):
        t = O.occgrid_times(1, 16, (0, 0, 0, 1, 1, 1), 9, 0, j).astype(np.float64)
        c = np.stack([0.3 + 0.4 * t, np.full_like(t, 0.5), np.full_like(t, 0.5)], 1)
        v = np.where(np.linalg.norm(xyz - c, axis=1) < 0.2, 2.0, 0.0).astype(np.float32)
        ref = v if ref is None else np.maximum(ref, v)
    assert np.array_equal(a, ref) and ref.max() == 2.0
