"""One C4 particle-Gibbs sweep (64 chains, K=2^12, N=512) for ncu launch lists."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
e = Engine(0)
K, N, B = 4096, 512, 64
ys = np.asarray(models.sv(K - 1).arrays["y"], np.float64)
prior = abi.SvPrior(-1.0, 1.0, 2.0, 0.2, 0.05)
theta = np.ascontiguousarray(np.tile([-1.0, 0.9, 0.1], (B, 1)))
stars = np.ascontiguousarray(np.full((B, K), -1.0))
seeds = np.arange(B, dtype=np.uint64) + 1000
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for s in range(reps):
    t0 = time.perf_counter()
    e.sv_pgibbs_sweep(ys, theta, stars, seeds, prior, N, s)
    print("sweep", s, (time.perf_counter() - t0) * 1e3, "ms", flush=True)
