"""FP32 vs FP64 resampling law at full size: for each of
NSEED seeds per arm, one C5 run (K = 2^20, N = 1024, d = 4, multinomial) in the
FP32 throughput path and one in the FP64 parity path; per run the summary
statistics against the exact Kalman/RTS smoother (median / mean variance
ratio, rms z, mean z, log Z - exact). Prints one JSON object per run and a
Welch t per statistic. Usage: python tools/c5_law.py [config] [nseed]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2202_02264_b200 import abi  # noqa: E402
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "c5"
nseed = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = bench.CONFIGS[cname]
m = bench.build_model(cfg)
km, kP, ll = kalman_smooth(m)
sd = np.sqrt(np.einsum("tii->ti", kP))
e = Engine(0)
h = e.upload(m)
K, d = cfg["K"], m.d
stats = {"fp32": [], "fp64": []}
for prec, name in ((abi.FP32, "fp32"), (abi.FP64_PARITY, "fp64")):
    for seed in range(1, nseed + 1):
        t0 = time.perf_counter()
        e.smooth_resident(h, cfg["N"], abi.MULTINOMIAL, seed=1000 + seed, precision=prec)
        mean, cov, lz = e.resident_results(K, d)
        wall = time.perf_counter() - t0
        z = (mean - km) / sd
        vr = np.einsum("tii->ti", cov) / np.einsum("tii->ti", kP)
        row = dict(prec=name, seed=seed, mean_z=float(z.mean()), rms_z=float(np.sqrt((z ** 2).mean())),
                   med_vr=float(np.median(vr)), mean_vr=float(vr.mean()),
                   dlogz=float(lz - ll), wall_s=wall)
        stats[name].append(row)
        print(json.dumps(row), flush=True)
out = {}
for key in ("mean_z", "rms_z", "med_vr", "mean_vr", "dlogz"):
    a = np.array([r[key] for r in stats["fp32"]])
    b = np.array([r[key] for r in stats["fp64"]])
    t = (a.mean() - b.mean()) / np.sqrt(a.var(ddof=1) / len(a) + b.var(ddof=1) / len(b))
    out[key] = dict(fp32=float(a.mean()), fp32_se=float(a.std(ddof=1) / np.sqrt(len(a))),
                    fp64=float(b.mean()), fp64_se=float(b.std(ddof=1) / np.sqrt(len(b))),
                    welch_t=float(t))
print(json.dumps({"summary": out, "config": cname, "nseed": nseed}))
