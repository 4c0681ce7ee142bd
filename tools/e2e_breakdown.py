"""Where does the end-to-end (host arrays in, host moments out) time go?"""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2202_02264_b200.dsmc import Engine
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
m = bench.build_model(cfg, pinned=True)
e = Engine(0)
N = cfg["N"]
def wall(f, n=3):
    ts = []
    for _ in range(n):
        e.sync(); t0 = time.perf_counter(); f(); e.sync(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3
import torch
mo = torch.empty((cfg["K"], m.d), dtype=torch.float64, pin_memory=True).numpy()
co = torch.empty((cfg["K"], m.d, m.d), dtype=torch.float64, pin_memory=True).numpy()
e.smooth(m, N, 0, seed=1)
print("smooth (e2e)      ms", wall(lambda: e.smooth(m, N, 0, seed=2)))
print("smooth pinned out ms", wall(lambda: e.smooth(m, N, 0, seed=2, mean_out=mo, cov_out=co)))
h = e.upload(m); e.sync()
print("upload+prep       ms", wall(lambda: e.free_model(e.upload(m))))
print("resident run      ms", wall(lambda: e.smooth_resident(h, N, 0, seed=3)))
print("results D2H       ms", wall(lambda: e.resident_results(cfg["K"], m.d)))
print("timings", e.timings())
