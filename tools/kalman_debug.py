import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2202_02264_b200 import models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
if len(sys.argv) > 1 and sys.argv[1] == "dump":  # arrays for tools/kalman_scan_check.cu
    m = models.cv_tracking(1)
    for k in ["F", "b", "Q", "H", "R", "y", "m0", "P0"]:
        np.asarray(m.arrays[k], np.float64).ravel().tofile(k)
    sys.exit(0)
e = Engine(0)
for T in (0, 1, 5, 31, 32, 33, 63, 64, 100, 1023, 1024, 1025, 2000, 3000):
    for mk, name in ((lambda T: models.cv_tracking(T), "cv"), (lambda T: models.lgssm_check(T), "lg")):
        m = mk(T)
        hm, hP, hll = kalman_smooth(m)
        try:
            dm, dP, dll = e.kalman_smooth(m)
            print(name, T, "ok", np.abs(dm - hm).max(), np.abs(dP - hP).max(), dll - hll, flush=True)
        except Exception as ex:
            print(name, T, "ERR", ex, flush=True)
