"""The NACC_DEBUG build (libnacc_debug.so, csrc/debug.cu): device preconditions the
release build leaves to the caller -- unit directions (reading #8), σ >= 0,
ascending non-overlapping intervals inside the arrays, α in [0, 1], ascending
resampling edges -- are checked and reported as NACC_ERR_INVALID_ARGUMENT; valid inputs pass.
Runs in a subprocess because the library choice is made at import time (NACC_DEBUG=1)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2305_04966_b200 as N
from paper_2305_04966_b200 import _lib as L
assert L.LIB_PATH.endswith("libnacc_debug.so"), L.LIB_PATH

def bad(fn, what):
    try:
        fn()
    except N.NaccError as e:
        assert e.status == L.NACC_ERR_INVALID_ARGUMENT and "precondition" in str(e), str(e)
        print("rejected:", what)
        return
    raise AssertionError("accepted: " + what)

dev = torch.device("cuda")
grid = N.GridSpec(roi=(0, 0, 0, 1, 1, 1), res=8, levels=1)
bits = N.prepare_bits(grid, torch.full((16,), -1, dtype=torch.int32, device=dev))
o = torch.tensor([[0.5, 0.5, -0.5], [-0.5, 0.5, 0.5]], device=dev)
d = torch.tensor([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]], device=dev)
s = N.sampling_occgrid(o, d, grid, bits, N.MarchParams(step=0.01))  # valid
assert s.n_samples > 100
bad(lambda: N.sampling_occgrid(o, d * 1.5, grid, bits, N.MarchParams(step=0.01)), "non-unit direction")
sig = torch.ones(s.n_samples, device=dev)
N.filter_early_stop(s, sig, 1e-4)  # valid
sig_bad = sig.clone(); sig_bad[7] = -1.0
bad(lambda: N.filter_early_stop(s, sig_bad, 1e-4), "negative sigma")
rgb = torch.rand(s.n_samples, 3, device=dev)
N.render_fwd(s, sig, rgb, 1e-4)  # valid
t0 = s.t0.clone(); t0[5] = s.t1[5] + 0.5  # interval 5 ends before it starts / overlaps 6
s_bad = N.PackedSamples(s.packed_info, t0, s.t1, s.ray_id)
bad(lambda: N.render_fwd(s_bad, sig, rgb, 1e-4), "overlapping intervals")
pk_bad = s.packed_info.clone(); pk_bad[1, 1] += 5  # run past the end of the arrays
bad(lambda: N.render_fwd(N.PackedSamples(pk_bad, s.t0, s.t1, s.ray_id), sig, rgb, 1e-4), "run past the arrays")
alpha = torch.rand(s.n_samples, device=dev)
N.render_weights_alpha(s, alpha)  # valid
alpha_bad = alpha.clone(); alpha_bad[3] = 1.5
bad(lambda: N.render_weights_alpha(s, alpha_bad), "alpha > 1")
e = torch.linspace(0, 1, 33, device=dev).repeat(4, 1).contiguous()
N.importance_sample(e, 8, sigma=torch.rand(4, 32, device=dev))  # valid
e_bad = e.clone(); e_bad[2, 10] = 0.9
bad(lambda: N.importance_sample(e_bad, 8, sigma=torch.rand(4, 32, device=dev)), "descending edges")
print("debug build ok")
'''


def test_debug_build_checks_device_preconditions():
    import __graft_entry__

    __graft_entry__.build()
    env = dict(os.environ, NACC_DEBUG="1")
    r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "debug build ok" in r.stdout and r.stdout.count("rejected:") == 6
