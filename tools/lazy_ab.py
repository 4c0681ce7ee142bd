"""Bitwise A/B of two engine builds on the lazy samplers (MH and rejection):
python tools/lazy_ab.py run LIB OUT.npz ; python tools/lazy_ab.py cmp A B"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "run":
    import paper_2202_02264_b200.dsmc as D
    D.LIB_PATH = sys.argv[2]
    from paper_2202_02264_b200 import abi, models
    e = D.Engine(0)
    out = {}
    for name, m, N, rs, B in [("sv_mh", models.sv(1023), 512, abi.MH_LAZY, 16),
                              ("cv_mh", models.cv_tracking(511), 256, abi.MH_LAZY, 16),
                              ("crw_rej", models.constrained_rw(511, 0.3), 256, abi.REJECTION_LAZY, 16),
                              ("lg_mh", models.lgssm_check(1000), 300, abi.MH_LAZY, 16),
                              ("sv_mh13", models.sv(255), 200, abi.MH_LAZY, 13),
                              ("cv_mh2", models.cv_tracking(127), 128, abi.MH_LAZY, 2)]:
        r = e.smooth(m, N, rs, seed=7, precision=abi.FP32, want_pairs=True, mh_steps=B)
        out[name + "_l"] = r["pair_left"]
        out[name + "_r"] = r["pair_right"]
        out[name + "_ev"] = np.array([r["weight_evals"]])
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
