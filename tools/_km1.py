import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2604_23150_b200 import moeplace as mp, policies as pol
R, E, K = 65536, 128, 4
rng = np.random.default_rng(0)
dom = rng.integers(0, K, R)
pref = np.stack([rng.choice(E, 32, replace=False) for _ in range(K)])
X = rng.poisson(0.3, (R, E)).astype(np.float64)
for r in range(R):
    X[r, pref[dom[r]]] += rng.poisson(2.0, 32)
X[X.sum(1) == 0, 0] = 1.0
eng = mp.Engine(0)
d = pol.l2_normalize_rows_device(eng, torch.from_numpy(X))
for s in [1, 4]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = pol.kmeans_device(eng, d, R, E, K, s, 100, 1e-6)
    print(s, m.iterations_run, round(time.perf_counter() - t0, 4))
