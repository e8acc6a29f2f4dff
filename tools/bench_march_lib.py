"""Shared timing helper of the tools/bench_*.py scripts."""
import numpy as np
import torch


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
