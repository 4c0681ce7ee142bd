"""Replay the SV particle-Gibbs failure of the tensor-core pass 1: run the
tests/test_gpu_pgibbs.py loop, save the state before the failing sweep,
re-run it (determinism) and per chain (which chains fail)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200.dsmc import Engine
from tests.test_gpu_pgibbs import _data, _prior

e = Engine(0)
T, B, N = 511, 64, 256
ys = _data(T, seed=90210)
mode = sys.argv[1]
if mode == "find":
    theta = np.ascontiguousarray(np.tile([-0.5, 0.8, 0.2], (B, 1)))
    stars = np.ascontiguousarray(np.full((B, T + 1), -1.0))
    seeds = np.arange(B, dtype=np.uint64) + 1000
    for s in range(60):
        th0, st0 = theta.copy(), stars.copy()
        try:
            e.sv_pgibbs_sweep(ys, theta, stars, seeds, _prior(), N, s)
        except Exception as ex:
            print("sweep", s, "failed:", ex)
            np.savez("gpurun_out/tc_fail.npz", theta=th0, stars=st0, sweep=s)
            break
    else:
        print("no failure")
        sys.exit(0)
d = np.load("gpurun_out/tc_fail.npz")
s = int(d["sweep"])
seeds = np.arange(B, dtype=np.uint64) + 1000
for rep in range(2):
    th, st = d["theta"].copy(), d["stars"].copy()
    try:
        e.sv_pgibbs_sweep(ys, th, st, seeds, _prior(), N, s)
        print(os.environ.get("DSMC_PAIR_KERNEL", "tc"), "replay", rep, "ok")
    except Exception as ex:
        print(os.environ.get("DSMC_PAIR_KERNEL", "tc"), "replay", rep, "failed:", ex)
bad = []
for b in range(B):
    th = np.ascontiguousarray(d["theta"][b:b + 1].copy())
    st = np.ascontiguousarray(d["stars"][b:b + 1].copy())
    try:
        e.sv_pgibbs_sweep(ys, th, st, seeds[b:b + 1], _prior(), N, s)
    except Exception as ex:
        bad.append(b)
print("failing chains", bad, [tuple(np.round(d["theta"][b], 4)) for b in bad])
