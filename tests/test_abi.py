"""CPU tests of the boundary: the C-ABI library loads and exports every
symbol include/dsmc_b200.h declares; host-side pieces that need no GPU
(the Kalman proposal builder) agree with an independent numpy restatement;
the product fails loudly without a device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dsmc_b200.h")
LIB = os.path.join(ROOT, "paper_2202_02264_b200", "libdsmc_b200.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"DSMC_API\s+[\w\s\*]+?\b(dsmc_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["dsmc_create", "dsmc_smooth", "dsmc_resample_table", "dsmc_conditional_sweep",
              "dsmc_sv_pgibbs_sweep", "dsmc_smooth_resident", "dsmc_kalman_smooth",
              "dsmc_ffbs_smooth", "dsmc_make_leaf", "dsmc_resample_blocks",
              "dsmc_resample_indices", "dsmc_lazy_begin", "dsmc_lazy_probes", "dsmc_lazy_answer",
              "dsmc_lazy_finish", "dsmc_kalman_smooth_device", "dsmc_model_upload_window"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: make -C paper_2202_02264_b200/csrc"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dsmc_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        getattr(lib, s)


def test_library_has_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def numpy_rts(m):
    """Independent restatement of kalman.cpp:78-138 (numpy, no Joseph form)."""
    A = m.arrays
    K, d, dy = m.horizon + 1, m.d, m.dy
    F = A["F"].reshape(-1, d, d)
    Q = A["Q"].reshape(-1, d, d)
    H = A["H"].reshape(-1, dy, d)
    R = A["R"].reshape(-1, dy, dy)
    b = A["b"].reshape(-1, d)
    y = A["y"].reshape(K, dy)
    g = lambda X, t: X[t if len(X) > 1 else 0]
    fm, fP, pm, pP = [None] * K, [None] * K, [None] * K, [None] * K
    for t in range(K):
        if t == 0:
            pm[0], pP[0] = A["m0"].reshape(d), A["P0"].reshape(d, d)
        else:
            pm[t] = g(F, t) @ fm[t - 1] + g(b, t)
            pP[t] = g(F, t) @ fP[t - 1] @ g(F, t).T + g(Q, t)
        S = g(H, t) @ pP[t] @ g(H, t).T + g(R, t)
        Kg = pP[t] @ g(H, t).T @ np.linalg.inv(S)
        fm[t] = pm[t] + Kg @ (y[t] - g(H, t) @ pm[t])
        fP[t] = pP[t] - Kg @ S @ Kg.T
    sm, sP = [None] * K, [None] * K
    sm[-1], sP[-1] = fm[-1], fP[-1]
    for t in range(K - 2, -1, -1):
        G = fP[t] @ g(F, t + 1).T @ np.linalg.inv(pP[t + 1])
        sm[t] = fm[t] + G @ (sm[t + 1] - pm[t + 1])
        sP[t] = fP[t] + G @ (sP[t + 1] - pP[t + 1]) @ G.T
    return np.array(sm), np.array(sP)


@pytest.mark.parametrize("builder", [lambda: models.lgssm_check(60), lambda: models.cv_tracking(40)])
def test_kalman_proposals_match_numpy(builder):
    m = builder()
    sm, sP = numpy_rts(m)
    assert np.allclose(m.arrays["prop_mean"], sm, rtol=1e-9, atol=1e-9)
    assert np.allclose(m.arrays["prop_cov"], sP, rtol=1e-9, atol=1e-12)


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2202_02264_b200.dsmc import DsmcError, Engine
    with pytest.raises(DsmcError):
        Engine(0)


def test_descriptor_layout_matches_header():
    # the ctypes mirror must match the C struct layout
    assert ctypes.sizeof(abi.ModelDesc) == 4 * 4 + 8 * 2 + 16 * 5 + 8 * 4 + 8 * 3 + 8 * 8
    assert abi.SmoothOpts.inject_logw.offset == 48
