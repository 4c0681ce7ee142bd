"""Wall time of the sequential FFBS comparator vs dSMC on the device (the
paper's Fig. 2 comparison), same model / N, host arrays in and out."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
e = Engine(0)
for T, N in [(1023, 256), (4095, 512), (16383, 1024)]:
    m = models.cv_tracking(T)
    e.ffbs(m, N, seed=1); e.smooth(m, N, seed=1)
    t0 = time.perf_counter(); r = e.ffbs(m, N, seed=2); tf = time.perf_counter() - t0
    t0 = time.perf_counter(); s = e.smooth(m, N, seed=2); td = time.perf_counter() - t0
    print(f"CV d=4 K={T+1} N={N}: FFBS {tf*1e3:8.1f} ms  dSMC {td*1e3:7.1f} ms  ratio {tf/td:5.1f}", flush=True)
