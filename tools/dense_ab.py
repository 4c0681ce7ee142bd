"""Bitwise A/B of two engine builds on the dense FP32 path (multinomial and
systematic): python tools/dense_ab.py run LIB OUT.npz ; ... cmp A B"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "run":
    import paper_2202_02264_b200.dsmc as D
    D.LIB_PATH = sys.argv[2]
    from paper_2202_02264_b200 import abi, models
    e = D.Engine(0)
    out = {}
    for name, m, N, rs in [("cv", models.cv_tracking(1023), 1024, abi.MULTINOMIAL),
                           ("cv_sys", models.cv_tracking(255), 512, abi.SYSTEMATIC),
                           ("sv", models.sv(511), 512, abi.MULTINOMIAL),
                           ("lg_big", models.lgssm_check(63), 1500, abi.MULTINOMIAL),
                           ("lg_rag", models.lgssm_check(100), 100, abi.MULTINOMIAL)]:
        r = e.smooth(m, N, rs, seed=11, precision=abi.FP32, want_pairs=True)
        out[name + "_l"] = r["pair_left"]
        out[name + "_r"] = r["pair_right"]
        out[name + "_mean"] = r["mean"]
    np.savez(sys.argv[3], **out)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    ok = True
    for k in a.files:
        same = np.array_equal(a[k], b[k])
        ok &= same
        print(k, "identical" if same else "DIFFERENT")
    print("ALL IDENTICAL" if ok else "MISMATCH")
