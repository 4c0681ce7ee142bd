"""Does the FP32 path resample with the same law as the FP64 parity path?

Path degeneracy at the root of a deep tree (few distinct ancestors per time)
makes single-run smoothed variances collapse; the collapse is a property of
the algorithm, so both precisions must show the SAME amount of it. This runs
many seeds of the constant-velocity model (the C2/C5 family) at both
precisions and compares the per-run mean variance ratio (smoothed var / RTS
var), rms z of the means and log Z - exact, with Welch t statistics.

    python tools/fp32_law.py [K N reps] ...
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2202_02264_b200 import abi  # noqa: E402
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [4096, 64, 300, 65536, 256, 40]
e = Engine(0)
print("| K | N | reps | stat | FP32 mean (se) | FP64 mean (se) | Welch t |")
print("|---|---|---|---|---|---|---|")
for c in range(0, len(args), 3):
    K, N, reps = args[c:c + 3]
    cfg = dict(bench.CONFIGS["c2"], K=K, N=N)
    m = bench.build_model(cfg)
    km, kP, ll = kalman_smooth(m)
    sd = np.sqrt(np.einsum("tii->ti", kP))
    stats = {}
    for prec, name in ((abi.FP32, "fp32"), (abi.FP64_PARITY, "fp64")):
        rows = []
        for s in range(reps):
            r = e.smooth(m, N, abi.MULTINOMIAL, seed=7000 + s, precision=prec)
            z = (r["mean"] - km) / sd
            vr = np.einsum("tii->ti", r["cov"]) / np.einsum("tii->ti", kP)
            rows.append((vr.mean(), np.sqrt((z * z).mean()), r["log_norm_const"] - ll))
        stats[name] = np.array(rows)
    for q, label in enumerate(("mean var ratio", "rms z", "log Z - exact")):
        a, b = stats["fp32"][:, q], stats["fp64"][:, q]
        sa, sb = a.std(ddof=1) / np.sqrt(reps), b.std(ddof=1) / np.sqrt(reps)
        t = (a.mean() - b.mean()) / np.hypot(sa, sb)
        print(f"| {K} | {N} | {reps} | {label} | {a.mean():.4f} ({sa:.4f}) | "
              f"{b.mean():.4f} ({sb:.4f}) | {t:+.2f} |")
