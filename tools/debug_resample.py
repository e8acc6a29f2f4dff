import sys
sys.path.insert(0, '.')
import numpy as np, torch
import oracle as O
import paper_2305_04966_b200 as N
rng = np.random.default_rng(11)
n, m = 700, 40
e = np.sort(rng.uniform(0, 1, (n, m + 1)), axis=1).astype(np.float32)
e[:, 0], e[:, -1] = 0, 1
w = np.where(rng.random((n, m)) < 0.4, 0, rng.uniform(0, 1, (n, m)))
w[:5] = 0.0
cdf = np.concatenate([np.zeros((n, 1)), np.cumsum(w, 1)], 1).astype(np.float32)
sg, _ = N.importance_sample(torch.from_numpy(e).cuda(), 33, cdf=torch.from_numpy(cdf).cuda(), map_kind=N.MAP_IDENTITY, t_near=1.0, t_far=5.0)
sr, _ = O.importance_sample(e, 33, cdf=cdf, map_kind=0, t_near=1.0, t_far=5.0)
F = O.importance_cdf(e, cdf=cdf, map_kind=0, t_near=1.0, t_far=5.0)
sg = sg.cpu().numpy()
r = 492
np.set_printoptions(precision=8, linewidth=200)
print('e', e[r]); print('cdf', cdf[r]); print('F', F[r]); print('gpu', sg[r]); print('ref', sr[r])
bad = np.nonzero(np.abs(sg - sr) > 1e-4)
print('n bad', len(bad[0]), list(zip(bad[0][:20], bad[1][:20])))
