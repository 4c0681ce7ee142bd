"""Python binding of the B200 dSMC engine's C ABI (include/dsmc_b200.h).

Thin ctypes layer: every call goes to the in-tree CUDA library
(paper_2202_02264_b200/libdsmc_b200.so). There is no CPU fallback — if the
library is missing or no CUDA device is present, construction raises.
Errors map to the reference's exception classes (smoother.cpp / resampling.cpp
raise invalid_argument / runtime_error / domain_error / logic_error).
"""
import ctypes as C
import os

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdsmc_b200.so")
_lib = None


class DsmcError(RuntimeError):
    pass


_EXC = {
    abi.DSMC_E_INVALID_ARGUMENT: ValueError,      # std::invalid_argument
    abi.DSMC_E_RUNTIME: RuntimeError,             # std::runtime_error
    abi.DSMC_E_DOMAIN: ArithmeticError,           # std::domain_error
    abi.DSMC_E_LOGIC: AssertionError,             # std::logic_error
}


def load_library():
    """Load the CUDA engine; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `make -C paper_2202_02264_b200/csrc` "
                          "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, sz, i, u32, u64, dp = C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, C.c_uint64, C.POINTER(C.c_double)
    u32p, u64p, u8p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint8)
    ip = C.POINTER(C.c_int)
    sig = {
        "dsmc_create": (i, [i, C.POINTER(vp)]),
        "dsmc_destroy": (None, [vp]),
        "dsmc_last_error": (C.c_char_p, [vp]),
        "dsmc_kernel_launches": (u64, [vp]),
        "dsmc_smooth": (i, [vp, C.POINTER(abi.ModelDesc), C.POINTER(abi.SmoothOpts), C.POINTER(abi.SmoothOut)]),
        "dsmc_model_upload": (i, [vp, C.POINTER(abi.ModelDesc), C.POINTER(vp)]),
        "dsmc_model_free": (None, [vp, vp]),
        "dsmc_smooth_resident": (i, [vp, vp, C.POINTER(abi.SmoothOpts)]),
        "dsmc_resident_results": (i, [vp, dp, dp, dp, ip]),
        "dsmc_sync": (i, [vp]),
        "dsmc_stream": (vp, [vp]),
        "dsmc_last_timings": (i, [vp, dp, i]),
        "dsmc_resample_table": (i, [vp, i, dp, sz, sz, sz, i, C.c_double, u64, u32, u64,
                                    u32p, u32p, dp, ip, u64p, ip]),
        "dsmc_philox_blocks": (i, [vp, u64p, u64p, sz, u64p]),
        "dsmc_exp_w": (i, [vp, dp, sz, dp]),
        "dsmc_conditional_sweep": (i, [vp, C.POINTER(abi.ModelDesc), i, dp, u64p,
                                       C.POINTER(abi.CondOpts), u32, dp, u8p, dp, u64p]),
        "dsmc_kalman_smooth": (i, [C.POINTER(abi.ModelDesc), dp, dp, dp]),
        "dsmc_window_run": (i, [vp, vp, C.POINTER(abi.WindowOpts)]),
        "dsmc_window_boundary": (i, [vp, i, vp, vp, vp]),
        "dsmc_cross_combine": (i, [vp, vp, C.POINTER(abi.WindowOpts), i, i, C.c_longlong, vp, vp,
                                   vp, vp, vp, vp, vp, vp]),
        "dsmc_model_upload_window": (i, [vp, C.POINTER(abi.ModelDesc), i, i, C.POINTER(vp)]),
        "dsmc_kalman_smooth_device": (i, [vp, C.POINTER(abi.ModelDesc), dp, dp, dp]),
        "dsmc_window_remap": (i, [vp, i, vp]),
        "dsmc_window_finish": (i, [vp, vp, vp, vp]),
        "dsmc_ffbs_smooth": (i, [vp, C.POINTER(abi.ModelDesc), C.POINTER(abi.FfbsOpts), dp, dp,
                                 dp, dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if hasattr(lib, "dsmc_sv_pgibbs_sweep"):
        f = lib.dsmc_sv_pgibbs_sweep
        f.restype = i
        f.argtypes = [vp, i, i, dp, C.POINTER(abi.SvPrior), dp, dp, u64p, sz, i, u32, u8p, u64p]
    _lib = lib
    return lib


def kalman_smooth(model):
    """Exact RTS smoother of an LGSSM Model (host C++). -> (means, covs, loglik)."""
    lib = load_library()
    K, d = model.horizon + 1, model.d
    m = np.zeros((K, d))
    P = np.zeros((K, d, d))
    ll = C.c_double()
    rc = lib.dsmc_kalman_smooth(C.byref(model.desc), abi.dptr(m), abi.dptr(P), C.byref(ll))
    if rc:
        raise RuntimeError(f"dsmc_kalman_smooth failed ({rc})")
    return m, P, ll.value


class Engine:
    """One CUDA context (device + stream + memory arena)."""

    def __init__(self, device=0):
        self.lib = load_library()
        self.ctx = C.c_void_p()
        rc = self.lib.dsmc_create(device, C.byref(self.ctx))
        if rc:
            raise DsmcError(f"dsmc_create failed ({rc}): no CUDA device {device}")

    def close(self):
        if self.ctx:
            self.lib.dsmc_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            msg = self.lib.dsmc_last_error(self.ctx).decode()
            raise _EXC.get(rc, DsmcError)(msg)

    @property
    def launches(self):
        return int(self.lib.dsmc_kernel_launches(self.ctx))

    # ------------------------------------------------------------- probes
    def philox(self, ctr, key, n_blocks=1):
        c = (C.c_uint64 * 4)(*ctr)
        k = (C.c_uint64 * 2)(*key)
        out = np.zeros(4 * n_blocks, dtype=np.uint64)
        self._check(self.lib.dsmc_philox_blocks(self.ctx, c, k, n_blocks,
                                                out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def exp_w(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self.lib.dsmc_exp_w(self.ctx, abi.dptr(x), x.size, abi.dptr(out)))
        return out

    # ------------------------------------------------------- resampling
    def resample_table(self, resampler, logw, n_out, key, mh_steps=16, bound=None):
        """resample_pairs on a dense table (resampling.hpp:85-87)."""
        logw = np.ascontiguousarray(logw, dtype=np.float64)
        n = logw.shape[0]
        seed, level, node = key
        left = np.zeros(max(n_out, 1), dtype=np.uint32)
        right = np.zeros(max(n_out, 1), dtype=np.uint32)
        lmw = C.c_double()
        has = C.c_int()
        ev = C.c_uint64()
        biased = C.c_int()
        self._check(self.lib.dsmc_resample_table(
            self.ctx, resampler, abi.dptr(logw), n, n_out, mh_steps,
            0 if bound is None else 1, 0.0 if bound is None else float(bound),
            seed, level, node, abi.u32ptr(left), abi.u32ptr(right), C.byref(lmw),
            C.byref(has), C.byref(ev), C.byref(biased)))
        return dict(left=left[:n_out], right=right[:n_out],
                    log_mean_weight=lmw.value if has.value else None,
                    weight_evals=ev.value, biased=bool(biased.value))

    # --------------------------------------------------------- smoothing
    def smooth(self, model, n_particles, resampler=abi.MULTINOMIAL, seed=0,
               precision=abi.FP32, mh_steps=16, inject_states=None,
               inject_logw=None, want_paths=False, want_moments=True,
               want_pairs=False, want_leaves=False, mean_out=None, cov_out=None,
               want_leaf_logw=False):
        """run_smoother (smoother.hpp:128-129) on the GPU; host in/out.
        mean_out / cov_out: optional preallocated (e.g. pinned) host arrays of
        shape (K, d) / (K, d, d) that receive the moments."""
        K, d, N, T = model.horizon + 1, model.d, n_particles, model.horizon
        inj_x = None if inject_states is None else np.ascontiguousarray(inject_states, np.float64)
        inj_w = None if inject_logw is None else np.ascontiguousarray(inject_logw, np.float64)
        opts = abi.SmoothOpts(N, resampler, mh_steps, seed, precision,
                              abi.dptr(inj_x), abi.dptr(inj_w))
        res = {}
        paths = np.zeros((K, N, d)) if want_paths else None
        mean = (mean_out if mean_out is not None else np.zeros((K, d))) if want_moments else None
        cov = (cov_out if cov_out is not None else np.zeros((K, d, d))) if want_moments else None
        pl = np.zeros((max(T, 1), N), np.uint32) if want_pairs else None
        pr = np.zeros((max(T, 1), N), np.uint32) if want_pairs else None
        lmw = np.zeros(max(T, 1)) if want_pairs else None
        leaves = np.zeros((K, N, d)) if want_leaves else None
        leaf_lw = np.zeros((K, N)) if want_leaf_logw else None
        out = abi.SmoothOut(abi.dptr(paths), abi.dptr(mean), abi.dptr(cov),
                            abi.u32ptr(pl), abi.u32ptr(pr), abi.dptr(lmw),
                            abi.dptr(leaves), abi.dptr(leaf_lw))
        self._check(self.lib.dsmc_smooth(self.ctx, C.byref(model.desc), C.byref(opts), C.byref(out)))
        res.update(paths=paths, mean=mean, cov=cov,
                   pair_left=None if pl is None else pl[:T], pair_right=None if pr is None else pr[:T],
                   log_mean_weight=None if lmw is None else lmw[:T], leaves=leaves,
                   leaf_logw=leaf_lw,
                   log_norm_const=out.log_norm_const if out.has_log_norm_const else None,
                   levels=out.levels, weight_evals=out.weight_evals,
                   biased=bool(out.biased), wall_time_ms=out.wall_time_ms)
        return res

    def upload(self, model):
        h = C.c_void_p()
        self._check(self.lib.dsmc_model_upload(self.ctx, C.byref(model.desc), C.byref(h)))
        return h

    def free_model(self, h):
        self.lib.dsmc_model_free(self.ctx, h)

    def smooth_resident(self, handle, n_particles, resampler=abi.MULTINOMIAL, seed=0,
                        precision=abi.FP32, mh_steps=16):
        opts = abi.SmoothOpts(n_particles, resampler, mh_steps, seed, precision, None, None)
        self._check(self.lib.dsmc_smooth_resident(self.ctx, handle, C.byref(opts)))

    def resident_results(self, K, d):
        mean = np.zeros((K, d))
        cov = np.zeros((K, d, d))
        lnc = C.c_double()
        has = C.c_int()
        self._check(self.lib.dsmc_resident_results(self.ctx, abi.dptr(mean), abi.dptr(cov),
                                                   C.byref(lnc), C.byref(has)))
        return mean, cov, (lnc.value if has.value else None)

    def sync(self):
        self._check(self.lib.dsmc_sync(self.ctx))

    def stream_handle(self):
        return self.lib.dsmc_stream(self.ctx)

    def timings(self):
        """Device ms of the last resident run: leaves, levels, composition,
        pair kernels (sum), sample kernels (sum), number of pair launches."""
        ms = (C.c_double * 6)()
        n = self.lib.dsmc_last_timings(self.ctx, ms, 6)
        return list(ms[:n])

    def kalman_smooth(self, model):
        """Kalman/RTS on the device by parallel scans -> (means, covs, loglik)."""
        K, d = model.horizon + 1, model.d
        m, P, ll = np.zeros((K, d)), np.zeros((K, d, d)), C.c_double()
        self._check(self.lib.dsmc_kalman_smooth_device(self.ctx, C.byref(model.desc), abi.dptr(m),
                                                       abi.dptr(P), C.byref(ll)))
        return m, P, ll.value

    # ------------------------------------------------- time-sharded stages
    # Device buffers are passed as raw pointers (e.g. torch tensor data_ptr()
    # on the engine's stream); see paper_2202_02264_b200/sharded.py.
    def window_run(self, handle, n_particles, t0, length, seed, resampler=abi.MULTINOMIAL,
                   mh_steps=16):
        o = abi.WindowOpts(n_particles, resampler, mh_steps, seed, t0, length)
        self._check(self.lib.dsmc_window_run(self.ctx, handle, C.byref(o)))

    def upload_window(self, model, t0, length):
        """dsmc_model_upload_window: only the rows [t0 - 1, t0 + length] a
        time-sharded rank needs (its window and its right cross cut)."""
        h = C.c_void_p()
        self._check(self.lib.dsmc_model_upload_window(self.ctx, C.byref(model.desc), t0, length,
                                                      C.byref(h)))
        return h

    def window_boundary(self, side, d_states, d_col=None, d_root_lnc=None):
        """Enqueue the boundary slab gather and the root log Z copy (device
        pointers); no host synchronisation."""
        self._check(self.lib.dsmc_window_boundary(self.ctx, side, d_states, d_col, d_root_lnc))

    def cross_combine(self, handle, n_particles, seed, cut, level, node, d_xl, d_xr, d_colr,
                      d_lnc_l, d_lnc_r, d_l, d_r, d_lnc_out, resampler=abi.MULTINOMIAL,
                      mh_steps=16):
        o = abi.WindowOpts(n_particles, resampler, mh_steps, seed, 0, 2)
        self._check(self.lib.dsmc_cross_combine(self.ctx, handle, C.byref(o), cut, level, node,
                                                d_xl, d_xr, d_colr, d_lnc_l, d_lnc_r, d_l, d_r,
                                                d_lnc_out))

    def window_remap(self, side, d_idx):
        self._check(self.lib.dsmc_window_remap(self.ctx, side, d_idx))

    def window_finish(self, d_root_map, d_mean, d_cov):
        self._check(self.lib.dsmc_window_finish(self.ctx, d_root_map, d_mean, d_cov))

    # ------------------------------------------------------------- FFBS
    def ffbs(self, model, n_particles, n_draws=None, resampler=abi.MULTINOMIAL, seed=0,
             want_paths=False):
        """Sequential comparator: run_particle_filter + ffbs_sample
        (baselines.hpp:42-63) on the device, FP32. Returns per-time moments of
        the n_draws backward draws and the filter's log-likelihood."""
        K, d = model.horizon + 1, model.d
        M = n_particles if n_draws is None else n_draws
        mean, cov = np.zeros((K, d)), np.zeros((K, d, d))
        paths = np.zeros((M, K, d)) if want_paths else None
        ll = C.c_double()
        o = abi.FfbsOpts(n_particles, M, resampler, seed)
        self._check(self.lib.dsmc_ffbs_smooth(self.ctx, C.byref(model.desc), C.byref(o),
                                              abi.dptr(mean), abi.dptr(cov), abi.dptr(paths),
                                              C.byref(ll)))
        return dict(mean=mean, cov=cov, paths=paths, log_likelihood=ll.value)

    # --------------------------------------------------------- SV pGibbs
    def sv_pgibbs_sweep(self, ys, theta, stars, seeds, prior, n_particles, sweep,
                        resampler=abi.MULTINOMIAL):
        """One batched SV particle-Gibbs sweep (pgibbs_sweep, pgibbs.hpp:55-59):
        theta (B, 3) = (mu, phi, sigma2) and stars (B, T+1) are updated IN
        PLACE (float64, C-contiguous); returns (changed (B, T+1) bool, number
        of accepted phi moves)."""
        theta = np.asarray(theta)
        stars = np.asarray(stars)
        assert theta.dtype == np.float64 and theta.flags.c_contiguous
        assert stars.dtype == np.float64 and stars.flags.c_contiguous
        B, K = stars.shape
        ys = np.ascontiguousarray(ys, np.float64)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        changed = np.zeros((B, K), np.uint8)
        acc = C.c_uint64()
        self._check(self.lib.dsmc_sv_pgibbs_sweep(
            self.ctx, B, K - 1, abi.dptr(ys), C.byref(prior), abi.dptr(theta), abi.dptr(stars),
            seeds.ctypes.data_as(C.POINTER(C.c_uint64)), n_particles, resampler, sweep,
            abi.u8ptr(changed), C.byref(acc)))
        return changed.astype(bool), acc.value

    # ------------------------------------------------------- conditional
    def conditional_sweep(self, models, refs, seeds, n_particles, sweep,
                          resampler=abi.MULTINOMIAL, precision=abi.FP32,
                          inject_states=None):
        """run_conditional (conditional.hpp:48-51) batched over chains."""
        B = len(models)
        K, d = models[0].horizon + 1, models[0].d
        descs = (abi.ModelDesc * B)(*[m.desc for m in models])
        refs = np.ascontiguousarray(refs, dtype=np.float64).reshape(B, K, d)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        inj = None if inject_states is None else np.ascontiguousarray(inject_states, np.float64)
        opts = abi.CondOpts(n_particles, resampler, precision, abi.dptr(inj), None)
        out = np.zeros((B, K, d))
        changed = np.zeros((B, K), np.uint8)
        lnc = np.zeros(B)
        ev = np.zeros(B, np.uint64)
        self._check(self.lib.dsmc_conditional_sweep(
            self.ctx, descs, B, abi.dptr(refs), seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            C.byref(opts), sweep, abi.dptr(out), abi.u8ptr(changed), abi.dptr(lnc),
            ev.ctypes.data_as(C.POINTER(C.c_uint64))))
        return dict(paths=out, changed=changed.astype(bool), log_norm_const=lnc,
                    weight_evals=ev)
