"""Check that the CUDA-graph replay of the resident path reports the same
per-kernel timings (external event nodes) as eager launches, on C2."""
import sys, os
sys.path.insert(0, '.')
import bench
from paper_2202_02264_b200.dsmc import Engine
cfg = bench.CONFIGS["c2"]; m = bench.build_model(cfg)
e = Engine(0); h = e.upload(m)
for s in range(4):
    e.smooth_resident(h, 1024, 0, seed=s); e.sync(); print("run", s, e.timings(), e.launches)
