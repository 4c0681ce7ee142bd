"""Profiling driver: upload a config's model and run the resident smoothing
path `reps` times (no CPU work inside). Used under ncu."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2202_02264_b200.dsmc import Engine
from paper_2202_02264_b200 import abi
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="c2"); ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--precision", default="fp32")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
m = bench.build_model(cfg)
e = Engine(0); h = e.upload(m)
for r in range(a.reps):
    e.smooth_resident(h, cfg["N"], cfg["resampler"], seed=11 + r,
                      precision=abi.FP64_PARITY if a.precision == "fp64" else abi.FP32)
e.sync(); print("timings", e.timings())
