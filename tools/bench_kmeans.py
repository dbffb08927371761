"""K7 timing: request-clustering k-means on the GPU vs the host restatement
(bit-identical; 65,536 x 128, K=4, 10 restarts = 5.90 s CPU)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200 import policies as pol  # noqa: E402

R, E, K, restarts = 65536, 128, 4, 10
rng = np.random.default_rng(0)
dom = rng.integers(0, K, R)
pref = np.stack([rng.choice(E, 32, replace=False) for _ in range(K)])
X = rng.poisson(0.3, (R, E)).astype(np.float64)
for r in range(R):
    X[r, pref[dom[r]]] += rng.poisson(2.0, 32)
X[X.sum(1) == 0, 0] = 1.0
M = mp.ActivationMatrix(R, E, X, [f"d{d}" for d in dom])
eng = mp.Engine(0)
pol.run_cluster_stage(M, K, 99, 8, 1, engine=eng)  # warm-up (module load, scratch)
torch.cuda.synchronize()
dnorm = pol.l2_normalize_rows_device(eng, torch.from_numpy(X))
per = []
for sd in range(1, 1 + restarts):
    t0 = time.perf_counter()
    m = pol.kmeans_device(eng, dnorm, R, E, K, sd, 100, 1e-6)
    per.append((sd, m.iterations_run, round(time.perf_counter() - t0, 4)))
t0 = time.perf_counter()
dev = pol.run_cluster_stage(M, K, 1, 8, restarts, engine=eng)
t_dev = time.perf_counter() - t0
t0 = time.perf_counter()
host = pol.run_cluster_stage(M, K, 1, 8, restarts)
t_host = time.perf_counter() - t0
same = (dev.model.labels.tolist() == host.model.labels.tolist()
        and dev.model.objective == host.model.objective
        and np.array_equal(dev.model.centroids, host.model.centroids))
print(json.dumps({"rows": R, "dim": E, "K": K, "restarts": restarts,
                  "device_s": round(t_dev, 4), "host_s": round(t_host, 4),
                  "speedup": round(t_host / t_dev, 1), "bit_identical": same,
                  "objective": dev.model.objective, "per_restart_s_iters": per}))
