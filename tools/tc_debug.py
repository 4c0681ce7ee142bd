"""A/B check of the pass-1 kernels on one model: same seeds, log Z and means
under DSMC_PAIR_KERNEL=tc and =fma (run as two processes by the caller), plus
the SV particle-Gibbs loop of tests/test_gpu_pgibbs.py with the failing sweep
reported."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
from tests.test_gpu_pgibbs import _data, _prior

e = Engine(0)
for name, m, N in [("lg1", models.lgssm_check(255), 512), ("sv", models.sv(255), 512),
                   ("cv", models.cv_tracking(255), 1024), ("cox", models.cox(255), 512)]:
    r = e.smooth(m, N, abi.MULTINOMIAL, seed=3, precision=abi.FP32)
    print(os.environ.get("DSMC_PAIR_KERNEL", "tc"), name, "logZ %.6f" % r["log_norm_const"],
          "mean[0..3]", np.round(r["mean"][:3, 0], 4), flush=True)
T, B, N = 511, 64, 256
ys = _data(T, seed=90210)
theta = np.ascontiguousarray(np.tile([-0.5, 0.8, 0.2], (B, 1)))
stars = np.ascontiguousarray(np.full((B, T + 1), -1.0))
seeds = np.arange(B, dtype=np.uint64) + 1000
for s in range(60):
    th0 = theta.copy()
    try:
        e.sv_pgibbs_sweep(ys, theta, stars, seeds, _prior(), N, s)
    except Exception as ex:
        print("sweep", s, "failed:", ex)
        print("theta min", th0.min(0), "max", th0.max(0))
        break
else:
    print("60 sweeps ok; theta mean", theta.mean(0))
