import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2202_02264_b200 import models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth


def chk(e, m, tag):
    hm, hP, hll = kalman_smooth(m)
    try:
        dm, dP, dll = e.kalman_smooth(m)
        print(tag, "err", np.abs(dm - hm).max(), np.abs(dP - hP).max(), dll - hll, flush=True)
    except Exception as ex:
        print(tag, "EXC", ex, flush=True)


for seq in (["cv0", "cv1"], ["lg0", "cv1"], ["cv0", "lg0", "cv1"], ["cv1", "cv1"], ["cv5", "cv1", "cv5"]):
    e = Engine(0)
    for s in seq:
        m = models.cv_tracking(int(s[2:])) if s.startswith("cv") else models.lgssm_check(int(s[2:]))
        chk(e, m, "/".join(seq) + ": " + s)
    e.close()
