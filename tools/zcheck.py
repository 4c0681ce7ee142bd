"""Statistical check of the FP32 path vs exact RTS: mean z^2 over seeds (should be
~1/N_eff-scaled, equal for FP32 and FP64 parity)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
e = Engine(0)
for name, m in [("lgssm255", models.lgssm_check(255)), ("cv255", models.cv_tracking(255))]:
    km, kP, ll = kalman_smooth(m)
    sd = np.sqrt(np.einsum('tii->ti', kP))
    for N in (256, 1024, 2048):
        for prec in (abi.FP32, abi.FP64_PARITY):
            zs, lz = [], []
            for seed in range(12):
                r = e.smooth(m, N, abi.MULTINOMIAL, seed=1000 + seed, precision=prec)
                zs.append(np.mean(((r["mean"] - km) / sd) ** 2))
                lz.append(r["log_norm_const"] - ll)
            print(f"{name} N={N} prec={prec}: N*mean z^2 = {N*np.mean(zs):.2f} +- {N*np.std(zs)/np.sqrt(len(zs)):.2f}   "
                  f"logZ err mean {np.mean(lz):+.3f} sd {np.std(lz):.3f}", flush=True)
