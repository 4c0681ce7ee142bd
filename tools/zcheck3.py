"""test_cv_d4_means_match_kalman statistic over several 16-seed groups."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
e = Engine(0)
m = models.cv_tracking(127)
km, kP, ll = kalman_smooth(m)
for prec in [abi.FP32, abi.FP64_PARITY][:int(os.environ.get("NP", 2))]:
    for g in range(int(os.environ.get("G0", 0)), int(os.environ.get("G1", 5))):
        runs = [e.smooth(m, 1024, abi.MULTINOMIAL, seed=16 * g + s, precision=prec) for s in range(16)]
        means = np.stack([r["mean"] for r in runs])
        avg, se = means.mean(0), means.std(0, ddof=1) / 4
        z = (avg - km) / np.maximum(se, 1e-12)
        i = np.unravel_index(np.abs(z).argmax(), z.shape)
        print(f"prec={prec} group {g}: rms z {np.sqrt(np.mean(z**2)):.2f} max |z| {np.abs(z).max():.2f} at {i}", flush=True)
