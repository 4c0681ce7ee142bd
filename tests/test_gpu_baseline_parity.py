"""Bit-exact parity at the BASELINE configurations.

The compiled reference (oracle/_ref/libdsmc_ref.so: the reference's own
smoother.cpp / resampling.cpp / conditional.cpp built from /root/reference,
shipped prebuilt to the GPU box) runs the full-size workloads on the host with
all cores, and the device FP64 parity path must reproduce every ancestor index
of every combine, every root-path value, the weight-evaluation count and the
bias flag exactly, with log Z within 1e-12 relative (CUDA vs glibc `log`).

  C2  d = 4 constant-velocity LGSSM, K = 2^14, N = 1024, multinomial — both
      with the reference's leaves injected into the device and with the
      device's own FP64 leaves injected into the reference
      (smoother.cpp:226-277; test_smoother.cpp:292-341)
  C3  stochastic volatility, N = 4096, slices of the C3 trajectory: K = 2^12
      with MH-lazy (B = 16), K = 2^9 with rejection-lazy (resampling.cpp:
      233-324; the reference's scalar rejection loop needs ~350 trials per slot
      on the 2^10 slice, minutes of host time, so the exact sampler is pinned
      on the shorter slice)
  C4  conditional dSMC sweep of 64 chains x K = 2^12 x N = 512 (SV,
      multinomial; conditional.cpp:156-216)
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models

pytestmark = pytest.mark.gpu

C2_SEED = 1 + (1 << 32)  # experiment.cpp:42-45 salting of seed 1


def _threads():
    return len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def c2_model():
    from oracle.py import Oracle
    return models.cv_tracking((1 << 14) - 1, smoother=Oracle().kalman_smooth)


def _same_run(g, r, rs):
    assert np.array_equal(g["pair_left"], r["pair_left"]), "left ancestors differ"
    assert np.array_equal(g["pair_right"], r["pair_right"]), "right ancestors differ"
    assert np.array_equal(g["paths"], r["paths"]), "root paths differ"
    if r["log_norm_const"] is None:
        assert g["log_norm_const"] is None
    else:
        assert abs(g["log_norm_const"] - r["log_norm_const"]) <= 1e-12 * abs(r["log_norm_const"])
    assert g["weight_evals"] == r["weight_evals"]
    assert g["levels"] == r["levels"]
    assert g["biased"] == r["biased"]


def test_c2_full_size_bitwise_reference_leaves(engine, reference, c2_model):
    m, N = c2_model, 1024
    X, W = reference.leaves_all(m, N, C2_SEED)
    r = reference.run_injected(m, N, X, W, abi.MULTINOMIAL, seed=C2_SEED)
    g = engine.smooth(m, N, abi.MULTINOMIAL, seed=C2_SEED, precision=abi.FP64_PARITY,
                      inject_states=X, inject_logw=W, want_paths=True, want_pairs=True)
    _same_run(g, r, abi.MULTINOMIAL)
    assert r["weight_evals"] == ((1 << 14) - 1) * N * N
    # the device's own leaves (counter-addressed Philox + FP64 Box-Muller)
    # agree with the reference's glibc leaves to a few ulp
    d = engine.smooth(m, N, abi.MULTINOMIAL, seed=C2_SEED, precision=abi.FP64_PARITY,
                      want_leaves=True, want_moments=False)
    assert np.allclose(d["leaves"], X, rtol=1e-12, atol=1e-12)


def test_c2_full_size_bitwise_device_leaves(engine, reference, c2_model):
    """The other direction: leaves drawn on the device are fed to the
    reference (its proposal sampler replays them; its own weight callbacks
    weigh them) and the device reruns on the same (states, weights)."""
    m, N, seed = c2_model, 1024, 77
    d = engine.smooth(m, N, abi.MULTINOMIAL, seed=seed, precision=abi.FP64_PARITY,
                      want_leaves=True, want_leaf_logw=True, want_moments=False)
    Xd = d["leaves"]
    Wr = reference.leaf_weights(m, Xd)
    # the device's own (normalised) leaf weights vs the reference's weighting
    mx = Wr.max(1, keepdims=True)
    Wn = Wr - (mx + np.log(np.exp(Wr - mx).sum(1, keepdims=True)))
    assert np.allclose(d["leaf_logw"], Wn, rtol=0, atol=1e-11)
    r = reference.run_injected(m, N, Xd, Wr, abi.MULTINOMIAL, seed=seed)
    g = engine.smooth(m, N, abi.MULTINOMIAL, seed=seed, precision=abi.FP64_PARITY,
                      inject_states=Xd, inject_logw=Wr, want_paths=True, want_pairs=True)
    _same_run(g, r, abi.MULTINOMIAL)


def c3_slice(k):
    """The first 2^k times of the C3 trajectory (same data generator)."""
    ys = np.asarray(models.sv((1 << 16) - 1).arrays["y"], np.float64)[: 1 << k]
    return models.sv((1 << k) - 1, ys=ys)


@pytest.mark.parametrize("rs,k", [(abi.MH_LAZY, 12), (abi.REJECTION_LAZY, 9)])
def test_c3_lazy_n4096_bitwise(engine, reference, rs, k):
    m, N, seed = c3_slice(k), 4096, 3 + (2 << 32)
    X, W = reference.leaves_all(m, N, seed)
    r = reference.run_injected(m, N, X, W, rs, seed=seed, mh_steps=16)
    g = engine.smooth(m, N, rs, seed=seed, precision=abi.FP64_PARITY, mh_steps=16,
                      inject_states=X, inject_logw=W, want_paths=True, want_pairs=True)
    _same_run(g, r, rs)
    assert r["log_norm_const"] is None  # lazy: no log mean weight (smoother.cpp:220-222)
    if rs == abi.MH_LAZY:
        assert r["biased"] and r["weight_evals"] == ((1 << k) - 1) * N * 17


def test_c4_64_chains_full_shape_bitwise(engine, reference):
    """C4's conditional sweep at its full shape: 64 chains, K = 2^12, N = 512,
    each chain with its own seed and reference path; the device runs all 64
    chains in one batched sweep, the reference runs run_conditional per chain
    (chains over host threads, as experiment.cpp:618-642)."""
    K, N, B, sweep = 1 << 12, 512, 64, 5
    ys = np.asarray(models.sv(K - 1).arrays["y"], np.float64)
    m = models.sv(K - 1, mu=-1.0, phi=0.9, sigma=np.sqrt(0.1), ys=ys)
    rng = np.random.default_rng(2024)
    stars = -1.0 + 0.4 * np.cumsum(rng.standard_normal((B, K)), axis=1) / np.sqrt(K)
    seeds = [int(v) for v in 1000 + np.arange(B)]

    def ref_chain(c):
        X = reference.conditional_leaves_all(m, stars[c], N, seeds[c], sweep)
        return X, reference.conditional(m, stars[c], N, seeds[c], sweep)
    with ThreadPoolExecutor(max_workers=_threads()) as ex:
        outs = list(ex.map(ref_chain, range(B)))
    Xall = np.stack([o[0] for o in outs])
    g = engine.conditional_sweep([m] * B, stars[:, :, None], seeds, N, sweep,
                                 precision=abi.FP64_PARITY, inject_states=Xall)
    for c, (_, r) in enumerate(outs):
        assert np.array_equal(g["paths"][c, :, 0], r["path"][:, 0]), f"chain {c}"
        assert abs(g["log_norm_const"][c] - r["log_norm_const"]) <= \
            1e-12 * abs(r["log_norm_const"]), f"chain {c}"
        assert g["weight_evals"][c] == r["weight_evals"] == (K - 1) * (N * N + 1)
