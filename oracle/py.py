"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU checkers.

  Oracle()    oracle/liboracle.so — the plain-C restatement (dsmc_oracle.c)
  Reference() oracle/_ref/libdsmc_ref.so — the reference's own sources
              compiled from /root/reference (only where it was built)

Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
checker, never by the product path.
"""
import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2202_02264_b200 import abi  # noqa: E402  (struct layouts only)

ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libdsmc_ref.so")

_vp, _sz, _i, _u32, _u64 = C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, C.c_uint64
_dp, _u32p, _u64p, _ip = C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int)


class OracleError(RuntimeError):
    pass


_EXC = {abi.DSMC_E_INVALID_ARGUMENT: ValueError, abi.DSMC_E_RUNTIME: RuntimeError,
        abi.DSMC_E_DOMAIN: ArithmeticError, abi.DSMC_E_LOGIC: AssertionError}


def _u64arr(a):
    return (C.c_uint64 * len(a))(*a)


class _Base:
    def _check(self, rc):
        if rc:
            raise _EXC.get(rc, OracleError)(self._err())

    def philox(self, ctr, key):
        out = (C.c_uint64 * 4)()
        self._philox(_u64arr(ctr), _u64arr(key), out)
        return np.array(out[:], dtype=np.uint64)

    def stream(self, key, kind, n, substream=0):
        """kind: 'u64' | 'uniform' | 'uniform_pos' | 'normal'."""
        seed, level, node, role = key
        k = {"u64": 0, "uniform": 1, "uniform_pos": 2, "normal": 3}[kind]
        out = np.zeros(n, dtype=np.uint64 if k == 0 else np.float64)
        self._stream(seed, level, node, role, substream, k, n, out.ctypes.data_as(_vp))
        return out

    def resample_table(self, resampler, logw, n_out, key, mh_steps=16, bound=None):
        logw = np.ascontiguousarray(logw, dtype=np.float64)
        n = logw.shape[0]
        seed, level, node = key
        left = np.zeros(max(n_out, 1), np.uint32)
        right = np.zeros(max(n_out, 1), np.uint32)
        lmw, has, ev, biased = C.c_double(), C.c_int(), C.c_uint64(), C.c_int()
        self._check(self._resample(resampler, abi.dptr(logw), n, n_out, mh_steps,
                                   0 if bound is None else 1, 0.0 if bound is None else bound,
                                   seed, level, node, abi.u32ptr(left), abi.u32ptr(right),
                                   C.byref(lmw), C.byref(has), C.byref(ev), C.byref(biased)))
        return dict(left=left[:n_out], right=right[:n_out],
                    log_mean_weight=lmw.value if has.value else None,
                    weight_evals=ev.value, biased=bool(biased.value))


class Oracle(_Base):
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} not built (make -C oracle oracle)")
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.or_last_error.restype = C.c_char_p
        L.or_philox.argtypes = [_u64p, _u64p, _u64p]
        L.or_stream.argtypes = [_u64, _u32, _u64, _i, _u64, _i, _sz, _vp]
        L.or_exp_w.restype = C.c_double
        L.or_exp_w.argtypes = [C.c_double]
        L.or_reduce_sum.restype = C.c_double
        L.or_reduce_sum.argtypes = [_dp, _sz]
        L.or_log_sum_exp.restype = C.c_double
        L.or_log_sum_exp.argtypes = [_dp, _sz]
        L.or_exp_row_store.restype = C.c_double
        L.or_exp_row_store.argtypes = [_dp, _sz, C.c_double, _dp, _dp]
        L.or_resample_table.argtypes = [_i, _dp, _sz, _sz, _sz, _i, C.c_double, _u64, _u32,
                                        _u64, _u32p, _u32p, _dp, _ip, _u64p, _ip]
        L.or_build_schedule.argtypes = [_i, _ip]
        L.or_smooth.argtypes = [C.POINTER(abi.ModelDesc), C.POINTER(abi.SmoothOpts),
                                C.POINTER(abi.SmoothOut)]
        L.or_conditional.argtypes = [C.POINTER(abi.ModelDesc), _dp, _sz, _i, _u64, _u32,
                                     _dp, _dp, _dp, _dp, _ip, _u64p]
        L.or_sv_param_update.argtypes = [_dp, _i, C.POINTER(abi.SvPrior), _u64, _u32, _dp, _ip]
        L.or_gamma_draw.restype = C.c_double
        L.or_gamma_draw.argtypes = [C.c_double, C.c_double, _u64, _u32, _u64, _i]
        L.or_kalman_smooth.argtypes = [C.POINTER(abi.ModelDesc), _dp, _dp, _dp]
        self._philox = L.or_philox
        self._stream = L.or_stream
        self._resample = L.or_resample_table
        self._err = lambda: L.or_last_error().decode()

    def exp_w(self, x):
        return np.array([self.L.or_exp_w(float(v)) for v in np.ravel(x)])

    def schedule(self, horizon):
        pairs = np.zeros((max(horizon, 1), 5), np.int32)
        levels = self.L.or_build_schedule(horizon, pairs.ctypes.data_as(_ip))
        return levels, pairs[:horizon]

    def smooth(self, model, n_particles, resampler=abi.MULTINOMIAL, seed=0, mh_steps=16,
               inject_states=None, inject_logw=None, want_paths=True, want_pairs=True):
        K, d, N, T = model.horizon + 1, model.d, n_particles, model.horizon
        inj_x = None if inject_states is None else np.ascontiguousarray(inject_states, np.float64)
        inj_w = None if inject_logw is None else np.ascontiguousarray(inject_logw, np.float64)
        opts = abi.SmoothOpts(N, resampler, mh_steps, seed, abi.FP64_PARITY,
                              abi.dptr(inj_x), abi.dptr(inj_w))
        paths = np.zeros((K, N, d)) if want_paths else None
        mean = np.zeros((K, d))
        cov = np.zeros((K, d, d))
        pl = np.zeros((max(T, 1), N), np.uint32) if want_pairs else None
        pr = np.zeros((max(T, 1), N), np.uint32) if want_pairs else None
        lmw = np.zeros(max(T, 1)) if want_pairs else None
        leaves = np.zeros((K, N, d))
        out = abi.SmoothOut(abi.dptr(paths), abi.dptr(mean), abi.dptr(cov), abi.u32ptr(pl),
                            abi.u32ptr(pr), abi.dptr(lmw), abi.dptr(leaves), None)
        self._check(self.L.or_smooth(C.byref(model.desc), C.byref(opts), C.byref(out)))
        return dict(paths=paths, mean=mean, cov=cov,
                    pair_left=None if pl is None else pl[:T],
                    pair_right=None if pr is None else pr[:T],
                    log_mean_weight=None if lmw is None else lmw[:T], leaves=leaves,
                    log_norm_const=out.log_norm_const if out.has_log_norm_const else None,
                    levels=out.levels, weight_evals=out.weight_evals, biased=bool(out.biased))

    def conditional(self, model, ref, n_particles, seed, sweep, resampler=abi.MULTINOMIAL,
                    inject_states=None):
        K, d = model.horizon + 1, model.d
        ref = np.ascontiguousarray(ref, np.float64).reshape(K, d)
        inj = None if inject_states is None else np.ascontiguousarray(inject_states, np.float64)
        out = np.zeros((K, d))
        lnc, has, ev = C.c_double(), C.c_int(), C.c_uint64()
        self._check(self.L.or_conditional(C.byref(model.desc), abi.dptr(ref), n_particles,
                                          resampler, seed, sweep, abi.dptr(inj), None,
                                          abi.dptr(out), C.byref(lnc), C.byref(has), C.byref(ev)))
        return dict(path=out, log_norm_const=lnc.value if has.value else None,
                    weight_evals=ev.value)

    def kalman_smooth(self, model):
        """kalman.cpp:78-138 restated in C -> (means, covs, loglik)."""
        K, d = model.horizon + 1, model.d
        m, P, ll = np.zeros((K, d)), np.zeros((K, d, d)), C.c_double()
        self._check(self.L.or_kalman_smooth(C.byref(model.desc), abi.dptr(m), abi.dptr(P),
                                            C.byref(ll)))
        return m, P, ll.value

    def sv_param_update(self, path, theta, prior, seed, sweep):
        th = np.ascontiguousarray(theta, np.float64).copy()
        path = np.ascontiguousarray(path, np.float64)
        acc = C.c_int()
        self._check(self.L.or_sv_param_update(abi.dptr(path), len(path) - 1, C.byref(prior),
                                              seed, sweep, abi.dptr(th), C.byref(acc)))
        return th, bool(acc.value)


class Reference(_Base):
    """The compiled reference (only present where /root/reference was built)."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise ImportError(f"{REF_SO} not built (make -C oracle ref)")
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_philox.argtypes = [_u64p, _u64p, _u64p]
        L.ref_stream.argtypes = [_u64, _u32, _u64, _i, _u64, _i, _sz, _vp]
        L.ref_set_backend.argtypes = [_i]
        L.ref_exp_w.restype = C.c_double
        L.ref_exp_w.argtypes = [C.c_double]
        L.ref_vec_exp.argtypes = [_dp, _sz, _dp]
        L.ref_reduce_sum.restype = C.c_double
        L.ref_reduce_sum.argtypes = [_dp, _sz]
        L.ref_log_sum_exp.restype = C.c_double
        L.ref_log_sum_exp.argtypes = [_dp, _sz]
        L.ref_exp_row_store.restype = C.c_double
        L.ref_exp_row_store.argtypes = [_dp, _sz, C.c_double, _dp, _dp]
        L.ref_resample_table.argtypes = [_i, _dp, _sz, _sz, _sz, _i, C.c_double, _u64, _u32,
                                         _u64, _u32p, _u32p, _dp, _ip, _u64p, _ip]
        L.ref_build_schedule.argtypes = [_i, _ip, _ip]
        L.ref_tree_depth.argtypes = [_i]
        M = C.POINTER(abi.ModelDesc)
        L.ref_make_leaf.argtypes = [M, _i, _sz, _u64, _dp, _dp, _dp, _ip, _dp]
        L.ref_stitch_rows.argtypes = [M, _i, _dp, _dp, _sz, _dp]
        L.ref_stitch_weight.argtypes = [M, _i, _dp, _dp, _dp]
        L.ref_stitch_bound.argtypes = [M, _i, _dp]
        L.ref_run_smoother.argtypes = [M, _sz, _i, _sz, _u64, _i, _dp, _dp, _ip, _u64p, _ip,
                                       _ip, _dp]
        L.ref_trace_smoother.argtypes = [M, _sz, _i, _sz, _u64, _dp, _u32p, _u32p, _dp, _dp, _ip]
        L.ref_run_conditional.argtypes = [M, _dp, _sz, _i, _u64, _u32, _dp, _dp, _ip, _u64p]
        L.ref_conditional_leaf.argtypes = [M, _i, _sz, _u64, _u32, _dp, _dp, _dp]
        L.ref_run_injected.argtypes = [M, _sz, _i, _sz, _u64, _i, _dp, _dp, _dp, _u32p, _u32p,
                                       _dp, _dp, _ip, _u64p, _ip, _ip]
        L.ref_leaf_weights_all.argtypes = [M, _dp, _sz, _dp]
        L.ref_make_leaves_all.argtypes = [M, _sz, _u64, _i, _dp, _dp]
        L.ref_gamma_draw.argtypes = [C.c_double, C.c_double, _u64, _u32, _u64, _i, _dp]
        L.ref_sv_param_update.argtypes = [_dp, _i, C.POINTER(abi.SvPrior), _u64, _u32, _dp, _ip]
        L.ref_conditional_leaves_all.argtypes = [M, _sz, _u64, _u32, _dp, _dp]
        self._philox = L.ref_philox
        self._stream = L.ref_stream
        self._resample = L.ref_resample_table
        self._err = lambda: L.ref_last_error().decode()

    def set_backend(self, b):
        self._check(self.L.ref_set_backend(b))

    def leaves(self, model, n, seed):
        """make_leaf for every t: states, raw and normalised weights, flags."""
        K, d = model.horizon + 1, model.d
        X = np.zeros((K, n, d))
        raw = np.zeros((K, n))
        norm = np.zeros((K, n))
        uni = np.zeros(K, bool)
        lnc = np.zeros(K)
        for t in range(K):
            u, l = C.c_int(), C.c_double()
            x = np.zeros((n, d))
            r = np.zeros(n)
            w = np.zeros(n)
            self._check(self.L.ref_make_leaf(C.byref(model.desc), t, n, seed, abi.dptr(x),
                                             abi.dptr(r), abi.dptr(w), C.byref(u), C.byref(l)))
            X[t], raw[t], norm[t], uni[t], lnc[t] = x, r, w, bool(u.value), l.value
        return dict(states=X, raw_logw=raw, logw=norm, uniform=uni, lnc=lnc)

    def run_smoother(self, model, n, resampler=abi.MULTINOMIAL, seed=0, mh_steps=16,
                     threads=1, want_paths=True):
        K, d = model.horizon + 1, model.d
        paths = np.zeros((K, n, d)) if want_paths else None
        lnc, has, ev, lev, biased, wall = (C.c_double(), C.c_int(), C.c_uint64(), C.c_int(),
                                           C.c_int(), C.c_double())
        self._check(self.L.ref_run_smoother(C.byref(model.desc), n, resampler, mh_steps, seed,
                                            threads, abi.dptr(paths), C.byref(lnc), C.byref(has),
                                            C.byref(ev), C.byref(lev), C.byref(biased),
                                            C.byref(wall)))
        return dict(paths=paths, log_norm_const=lnc.value if has.value else None,
                    weight_evals=ev.value, levels=lev.value, biased=bool(biased.value),
                    wall_time_ms=wall.value)

    def run_injected(self, model, n, states, raw_logw=None, resampler=abi.MULTINOMIAL, seed=0,
                     mh_steps=16, threads=None, want_pairs=True, want_paths=True):
        """run_smoother on injected leaves (ref_run_injected), multithreaded."""
        K, d, T = model.horizon + 1, model.d, model.horizon
        X = np.ascontiguousarray(states, np.float64)
        W = None if raw_logw is None else np.ascontiguousarray(raw_logw, np.float64)
        assert X.shape == (K, n, d)
        paths = np.zeros((K, n, d)) if want_paths else None
        pl = np.zeros((max(T, 1), n), np.uint32) if want_pairs else None
        pr = np.zeros((max(T, 1), n), np.uint32) if want_pairs else None
        lmw = np.zeros(max(T, 1)) if want_pairs else None
        lnc, has, ev, lev, bi = C.c_double(), C.c_int(), C.c_uint64(), C.c_int(), C.c_int()
        threads = threads or len(os.sched_getaffinity(0))
        self._check(self.L.ref_run_injected(
            C.byref(model.desc), n, resampler, mh_steps, seed, threads, abi.dptr(X), abi.dptr(W),
            abi.dptr(paths), abi.u32ptr(pl), abi.u32ptr(pr), abi.dptr(lmw), C.byref(lnc),
            C.byref(has), C.byref(ev), C.byref(lev), C.byref(bi)))
        return dict(paths=paths, pair_left=None if pl is None else pl[:T],
                    pair_right=None if pr is None else pr[:T],
                    log_mean_weight=None if lmw is None else lmw[:T],
                    log_norm_const=lnc.value if has.value else None, weight_evals=ev.value,
                    levels=lev.value, biased=bool(bi.value))

    def gamma_draw(self, shape, rate, key):
        out = C.c_double()
        seed, level, node, role = key
        self._check(self.L.ref_gamma_draw(shape, rate, seed, level, node, role, C.byref(out)))
        return out.value

    def sv_param_update(self, path, theta, prior, seed, sweep):
        th = np.ascontiguousarray(theta, np.float64).copy()
        path = np.ascontiguousarray(path, np.float64)
        acc = C.c_int()
        self._check(self.L.ref_sv_param_update(abi.dptr(path), len(path) - 1, C.byref(prior),
                                               seed, sweep, abi.dptr(th), C.byref(acc)))
        return th, bool(acc.value)

    def leaves_all(self, model, n, seed, threads=None):
        """make_leaf for every t (multithreaded): states (K, n, d), raw weights (K, n)."""
        K, d = model.horizon + 1, model.d
        X, W = np.zeros((K, n, d)), np.zeros((K, n))
        threads = threads or len(os.sched_getaffinity(0))
        self._check(self.L.ref_make_leaves_all(C.byref(model.desc), n, seed, threads,
                                               abi.dptr(X), abi.dptr(W)))
        return X, W

    def conditional_leaves_all(self, model, ref, n, seed, sweep):
        K, d = model.horizon + 1, model.d
        ref = np.ascontiguousarray(ref, np.float64).reshape(K, d)
        X = np.zeros((K, n, d))
        self._check(self.L.ref_conditional_leaves_all(C.byref(model.desc), n, seed, sweep,
                                                      abi.dptr(ref), abi.dptr(X)))
        return X

    def leaf_weights(self, model, states):
        """leaf_weights (fk_model.cpp:101-112) for every time: raw (T+1) x n."""
        X = np.ascontiguousarray(states, np.float64)
        K, n = X.shape[:2]
        W = np.zeros((K, n))
        self._check(self.L.ref_leaf_weights_all(C.byref(model.desc), abi.dptr(X), n, abi.dptr(W)))
        return W

    def trace_smoother(self, model, n, resampler=abi.MULTINOMIAL, seed=0, mh_steps=16):
        K, d, T = model.horizon + 1, model.d, model.horizon
        paths = np.zeros((K, n, d))
        pl = np.zeros((max(T, 1), n), np.uint32)
        pr = np.zeros((max(T, 1), n), np.uint32)
        lmw = np.zeros(max(T, 1))
        lnc, has = C.c_double(), C.c_int()
        self._check(self.L.ref_trace_smoother(C.byref(model.desc), n, resampler, mh_steps, seed,
                                              abi.dptr(paths), abi.u32ptr(pl), abi.u32ptr(pr),
                                              abi.dptr(lmw), C.byref(lnc), C.byref(has)))
        return dict(paths=paths, pair_left=pl[:T], pair_right=pr[:T], log_mean_weight=lmw[:T],
                    log_norm_const=lnc.value if has.value else None)

    def stitch_rows(self, model, c, xl, xr):
        n = xl.shape[0]
        out = np.zeros((n, n))
        self._check(self.L.ref_stitch_rows(C.byref(model.desc), c,
                                           abi.dptr(np.ascontiguousarray(xl, np.float64)),
                                           abi.dptr(np.ascontiguousarray(xr, np.float64)),
                                           n, abi.dptr(out)))
        return out

    def conditional_leaves(self, model, ref, n, seed, sweep):
        """conditional_leaf for every t (slot 0 = ref)."""
        K, d = model.horizon + 1, model.d
        ref = np.ascontiguousarray(ref, np.float64).reshape(K, d)
        X = np.zeros((K, n, d))
        for t in range(K):
            x = np.zeros((n, d))
            w = np.zeros(n)
            self._check(self.L.ref_conditional_leaf(C.byref(model.desc), t, n, seed, sweep,
                                                    abi.dptr(np.ascontiguousarray(ref[t])),
                                                    abi.dptr(x), abi.dptr(w)))
            X[t] = x
        return X

    def conditional(self, model, ref, n, seed, sweep, resampler=abi.MULTINOMIAL):
        K, d = model.horizon + 1, model.d
        ref = np.ascontiguousarray(ref, np.float64).reshape(K, d)
        out = np.zeros((K, d))
        lnc, has, ev = C.c_double(), C.c_int(), C.c_uint64()
        self._check(self.L.ref_run_conditional(C.byref(model.desc), abi.dptr(ref), n, resampler,
                                               seed, sweep, abi.dptr(out), C.byref(lnc),
                                               C.byref(has), C.byref(ev)))
        return dict(path=out, log_norm_const=lnc.value if has.value else None,
                    weight_evals=ev.value)
