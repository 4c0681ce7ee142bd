"""ctypes mirror of include/dsmc_b200.h (plain data only — no library load).

Shared by the product wrapper (paper_2202_02264_b200.dsmc) and by the test
oracles (oracle/py.py), which implement the same C contract.
"""
import ctypes as C

import numpy as np

DSMC_OK = 0
DSMC_E_INVALID_ARGUMENT = 1
DSMC_E_RUNTIME = 2
DSMC_E_DOMAIN = 3
DSMC_E_LOGIC = 4
DSMC_E_CUDA = 5
DSMC_E_NO_DEVICE = 6

MULTINOMIAL, SYSTEMATIC, MH_LAZY, REJECTION_LAZY = 0, 1, 2, 3
RESAMPLERS = {"multinomial": 0, "systematic": 1, "mh-lazy": 2, "rejection-lazy": 3}

ROLE_LEAF_PROPOSAL = 1
ROLE_PAIR_RESAMPLE = 2
ROLE_STAR_SELECT = 3
ROLE_GIBBS_PARAM = 4
ROLE_DATA_SIM = 5

FP32, FP64_PARITY = 0, 1
MODEL_LGSSM, MODEL_SV, MODEL_COX, MODEL_CRW, MODEL_THETA = 1, 2, 3, 4, 5

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)


class ModelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("state_dim", C.c_int), ("obs_dim", C.c_int),
        ("horizon", C.c_int),
        ("m0", _dp), ("P0", _dp),
        ("F", _dp), ("F_stride", C.c_int64),
        ("b", _dp), ("b_stride", C.c_int64),
        ("Q", _dp), ("Q_stride", C.c_int64),
        ("H", _dp), ("H_stride", C.c_int64),
        ("R", _dp), ("R_stride", C.c_int64),
        ("y", _dp), ("has_obs", _u8p),
        ("prop_mean", _dp), ("prop_cov", _dp),
        ("sv_mu", C.c_double), ("sv_phi", C.c_double), ("sv_sigma2", C.c_double),
        ("par", C.c_double * 8),
    ]


class SmoothOpts(C.Structure):
    _fields_ = [
        ("n_particles", C.c_size_t), ("resampler", C.c_int),
        ("mh_steps", C.c_size_t), ("seed", C.c_uint64), ("precision", C.c_int),
        ("inject_states", _dp), ("inject_logw", _dp),
    ]


class SmoothOut(C.Structure):
    _fields_ = [
        ("paths", _dp), ("mean", _dp), ("cov", _dp),
        ("pair_left", _u32p), ("pair_right", _u32p),
        ("log_mean_weight", _dp), ("leaf_states", _dp), ("leaf_logw", _dp),
        ("log_norm_const", C.c_double), ("has_log_norm_const", C.c_int),
        ("levels", C.c_int), ("weight_evals", C.c_uint64), ("biased", C.c_int),
        ("wall_time_ms", C.c_double),
    ]


class CondOpts(C.Structure):
    _fields_ = [
        ("n_particles", C.c_size_t), ("resampler", C.c_int),
        ("precision", C.c_int), ("inject_states", _dp), ("inject_logw", _dp),
    ]


class WindowOpts(C.Structure):
    _fields_ = [
        ("n_particles", C.c_size_t), ("resampler", C.c_int), ("mh_steps", C.c_size_t),
        ("seed", C.c_uint64), ("t0", C.c_int), ("len", C.c_int),
    ]


class FfbsOpts(C.Structure):
    _fields_ = [("n_particles", C.c_size_t), ("n_draws", C.c_size_t),
                ("resampler", C.c_int), ("seed", C.c_uint64)]


class SvPrior(C.Structure):
    _fields_ = [
        ("mu_mean", C.c_double), ("mu_var", C.c_double),
        ("s2_shape", C.c_double), ("s2_rate", C.c_double),
        ("phi_step", C.c_double),
    ]


def dptr(a):
    """double* of a contiguous float64 array (or NULL for None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def u32ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def u8ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)


class Model:
    """Plain-data model + the ctypes descriptor that borrows its arrays.

    Keep the Model alive while its descriptor is in use.
    """

    def __init__(self, kind, horizon, state_dim=1, obs_dim=1, **arrays):
        self.kind = kind
        self.horizon = horizon
        self.d = state_dim
        self.dy = obs_dim
        self.arrays = {k: (None if v is None else np.ascontiguousarray(v, dtype=np.uint8 if k == "has_obs" else np.float64))
                       for k, v in arrays.items() if k not in ("sv", "par")}
        self.sv = arrays.get("sv", (0.0, 0.0, 1.0))
        par = tuple(arrays.get("par", ()))
        self.par = par + (0.0,) * (8 - len(par))
        self.strides = {}
        d, dy, K = state_dim, obs_dim, horizon + 1
        per = {"F": d * d, "b": d, "Q": d * d, "H": dy * d, "R": dy * dy}
        for k, sz in per.items():
            a = self.arrays.get(k)
            if a is None:
                self.strides[k] = 0
            else:
                self.strides[k] = sz if a.size == K * sz else 0
                if a.size not in (sz, K * sz):
                    raise ValueError(f"{k}: size {a.size} is neither {sz} nor {K * sz}")
        self._desc = None

    @property
    def desc(self):
        if self._desc is None:
            A = self.arrays
            g = lambda k: dptr(A.get(k))
            self._desc = ModelDesc(
                self.kind, self.d, self.dy, self.horizon,
                g("m0"), g("P0"), g("F"), self.strides["F"], g("b"), self.strides["b"],
                g("Q"), self.strides["Q"], g("H"), self.strides["H"],
                g("R"), self.strides["R"], g("y"), u8ptr(A.get("has_obs")),
                g("prop_mean"), g("prop_cov"), *self.sv, (C.c_double * 8)(*self.par))
        return self._desc
