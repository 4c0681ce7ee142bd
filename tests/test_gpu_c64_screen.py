"""FP64 pass 1's FP32 row-max screen (combine64.cuh c64_row, fast = 1) must
give the same double row max as the full FP64 scan, so every ancestor index,
path value and log Z of the FP64 parity path is bit-identical with the screen
on and off (DSMC_C64_SCREEN=0 forces the full scan). Covers every model class
of the FP64 fill (LGSSM d = 1..4, SV, Cox, constrained RW with its -inf
columns, theta-logistic) and the three leaf-weight modes (level 1 has both
leaves' weights, upper levels none)."""
import os

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from tests.test_gpu_stress import lg_model

pytestmark = pytest.mark.gpu


def _run(engine, m, N, rs, seed, screen):
    os.environ["DSMC_C64_SCREEN"] = "1" if screen else "0"
    try:
        return engine.smooth(m, N, rs, seed=seed, precision=abi.FP64_PARITY, mh_steps=4,
                             want_pairs=True, want_paths=True)
    finally:
        os.environ.pop("DSMC_C64_SCREEN", None)


CASES = [
    ("cv", lambda: models.cv_tracking(2047), 512),
    ("lg1", lambda: models.lgssm_check(1023), 256),
    ("lg2", lambda: lg_model(2, 255, seed=5), 300),
    ("lg3", lambda: lg_model(3, 255, seed=6), 257),
    ("sv", lambda: models.sv(1023), 256),
    ("cox", lambda: models.cox(511), 200),
    ("crw", lambda: models.constrained_rw(511), 200),
    ("theta", lambda: models.theta_logistic(255), 128),
]


@pytest.mark.parametrize("name,make,N", CASES, ids=[c[0] for c in CASES])
def test_screen_is_bit_identical(engine, name, make, N):
    m = make()
    for rs in (abi.MULTINOMIAL, abi.SYSTEMATIC):
        a = _run(engine, m, N, rs, 11, False)
        b = _run(engine, m, N, rs, 11, True)
        assert np.array_equal(a["pair_left"], b["pair_left"]), (name, rs)
        assert np.array_equal(a["pair_right"], b["pair_right"]), (name, rs)
        assert np.array_equal(a["paths"], b["paths"]), (name, rs)
        assert a["log_norm_const"] == b["log_norm_const"], (name, rs)
        assert a["weight_evals"] == b["weight_evals"]


def test_screen_c2_full_size(engine):
    """C2's whole FP64 run (d = 4, K = 2^14, N = 1024): screen on == off."""
    m = models.cv_tracking((1 << 14) - 1)
    a = _run(engine, m, 1024, abi.MULTINOMIAL, 3, False)
    b = _run(engine, m, 1024, abi.MULTINOMIAL, 3, True)
    assert np.array_equal(a["pair_left"], b["pair_left"])
    assert np.array_equal(a["pair_right"], b["pair_right"])
    assert a["log_norm_const"] == b["log_norm_const"]
