"""Rejection-lazy at C3 shape (SV, N = 4096) on prefixes of the C3
trajectory, FP64 parity path vs FP32 path: weight evaluations per slot (the
acceptance cost) or the error raised. Usage: python tools/rejection_diag.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_02264_b200 import abi, models  # noqa: E402
from paper_2202_02264_b200.dsmc import Engine  # noqa: E402

e = Engine(0)
ys_all = np.asarray(models.sv((1 << 16) - 1).arrays["y"], np.float64)
for k in (9, 10, 11, 12):
    m = models.sv((1 << k) - 1, ys=ys_all[: 1 << k])
    for prec, name in ((abi.FP64_PARITY, "fp64"), (abi.FP32, "fp32")):
        try:
            r = e.smooth(m, 4096, abi.REJECTION_LAZY, seed=5, precision=prec)
            out = dict(k=k, prec=name, evals_per_slot=r["weight_evals"] / ((1 << k) - 1) / 4096)
        except Exception as ex:  # noqa: BLE001
            out = dict(k=k, prec=name, error=str(ex))
        print(json.dumps(out), flush=True)
y = ys_all[:1 << 12]
idx = np.argsort(np.abs(y))[:8]
print(json.dumps({"smallest_abs_y": [[int(i), float(y[i])] for i in idx]}))
