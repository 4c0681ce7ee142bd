"""Full-size accuracy of the headline run: C5 (K = 2^20, N = 1024, d = 4,
FP32, multinomial) smoothed means against the exact Kalman/RTS smoother, in
posterior standard deviations, plus log Z against the exact marginal
likelihood. Prints a markdown summary (profiles/r01h_c5_accuracy.md)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2202_02264_b200 import abi
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth

cname = sys.argv[1] if len(sys.argv) > 1 else "c5"
precs = [abi.FP32] if len(sys.argv) <= 2 else [abi.FP32, abi.FP64_PARITY]
nseed = int(os.environ.get("NSEED", "2"))
cfg = bench.CONFIGS[cname]
m = bench.build_model(cfg)
t0 = time.perf_counter()
km, kP, ll = kalman_smooth(m)
tk = time.perf_counter() - t0
e = Engine(0)
rows = []
for seed, prec in [(sd_, p_) for p_ in precs for sd_ in range(1, nseed + 1)]:
    r = e.smooth(m, cfg["N"], abi.MULTINOMIAL, seed=seed, precision=prec)
    sd = np.sqrt(np.einsum("tii->ti", kP))
    z = (r["mean"] - km) / sd
    vr = np.einsum("tii->ti", r["cov"]) / np.einsum("tii->ti", kP)
    rows.append((f"{seed} {'fp32' if prec == abi.FP32 else 'fp64'}", z, vr, r["log_norm_const"]))
print(f"# {cname} accuracy (K = {cfg['K']}, N = {cfg['N']}, d = {m.d})\n")
print(f"Exact Kalman/RTS on the host ({tk:.1f} s) vs two device runs of the headline "
      "configuration (`tools/c5_accuracy.py`). z = (smoothed mean - RTS mean) / RTS sd per "
      "time and component; variance ratio = smoothed var / RTS var.\n")
print("| seed / precision | mean z | rms z | max abs z | frac abs z > 4 | median var ratio | mean var ratio | log Z - exact |")
print("|---|---|---|---|---|---|---|---|")
for seed, z, vr, lz in rows:
    print(f"| {seed} | {z.mean():+.4f} | {np.sqrt((z**2).mean()):.4f} | {np.abs(z).max():.2f} | "
          f"{(np.abs(z) > 4).mean():.2e} | {np.median(vr):.4f} | {vr.mean():.4f} | {lz - ll:+.3f} |")
print(f"\nexact log-likelihood {ll:.3f}; the dSMC estimate of log Z carries O(sqrt(T)/N) "
      "Monte Carlo noise and a small negative (Jensen) bias.")
