import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
e = Engine(0)
m = models.lgssm_check(255)
km, kP, ll = kalman_smooth(m)
sd = np.sqrt(np.einsum('tii->ti', kP))
for N in (1024, 2048):
    for prec in (abi.FP32, abi.FP64_PARITY):
        mx, mz = [], []
        for seed in range(40):
            r = e.smooth(m, N, abi.MULTINOMIAL, seed=seed, precision=prec)
            z = (r["mean"] - km) / sd
            mx.append(np.abs(z).max()); mz.append(np.mean(z ** 2))
        mx = np.array(mx); mz = np.array(mz)
        print(f"N={N} prec={prec}: max|z| median {np.median(mx):.3f} p90 {np.percentile(mx,90):.3f} max {mx.max():.3f} (seed {mx.argmax()}) | N*mean z^2 mean {N*mz.mean():.2f} max {N*mz.max():.2f}", flush=True)
