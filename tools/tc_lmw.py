"""Pass-1 numerics A/B: level-1 log mean weights (inputs identical for both
kernels: the leaves) under DSMC_PAIR_KERNEL=tc / fma.
  python tools/tc_lmw.py run OUT.npz ; python tools/tc_lmw.py cmp A.npz B.npz"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models

CASES = lambda: [("lg1", models.lgssm_check(511), 512), ("sv", models.sv(511), 512),
                 ("sv_tiny", models.sv(511, sigma=0.057), 256), ("cv", models.cv_tracking(511), 1024),
                 ("cox", models.cox(511), 512), ("crw", models.constrained_rw(511), 256),
                 ("theta", models.theta_logistic(511), 256)]
if sys.argv[1] == "run":
    from paper_2202_02264_b200.dsmc import Engine
    e = Engine(0)
    out = {}
    for name, m, N in CASES():
        try:
            r = e.smooth(m, N, abi.MULTINOMIAL, seed=5, precision=abi.FP32, want_pairs=True)
            out[name] = r["log_mean_weight"][: (m.horizon + 1) // 2]
        except Exception as ex:
            print(name, "failed", ex)
    np.savez(sys.argv[2], **out)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        x, y = a[k], b[k] if k in b.files else None
        if y is None:
            print(k, "missing in", sys.argv[3]); continue
        d = np.abs(x - y)
        print(f"{k:8s} level-1 LMW max|diff| {np.nanmax(d):.3e} at {int(np.nanargmax(d))} "
              f"nonfinite {int((~np.isfinite(x)).sum())}/{int((~np.isfinite(y)).sum())}")
