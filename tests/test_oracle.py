"""CPU tests: the oracle restatement pinned against golden vectors and, where
it was built, the compiled reference itself. No GPU needed."""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi
from tests.cases import CASES, TABLES, table
from tests.conftest import golden_model


def test_philox_known_answers(oracle):
    # test_rng.cpp:32-47
    z = oracle.philox([0, 0, 0, 0], [0, 0])
    assert [int(v) for v in z] == [0x16554D9ECA36314C, 0xDB20FE9D672D0FDC,
                                   0xD7E772CEE186176B, 0x7E68B68AEC7BA23B]
    w = oracle.philox([0xDEADBEEF, 1, 2, 3], [0x9E3779B97F4A7C15, 0x243F6A8885A308D3])
    assert [int(v) for v in w] == [0x89AA73BBE8E9EBDB, 0x42065F627A6E7CCF,
                                   0xF103FF19821DA020, 0x0CF1B816FDC3EB80]


@pytest.mark.parametrize("kind", ["u64", "uniform", "uniform_pos", "normal"])
def test_streams_match_golden(oracle, golden, kind):
    got = oracle.stream((42, 3, 17, abi.ROLE_PAIR_RESAMPLE), kind, 257, substream=5)
    assert np.array_equal(got, golden[f"stream_{kind}"])


def test_exp_w_bit_identical_to_reference_scalar(oracle, golden):
    got = oracle.exp_w(golden["expw_x"])
    assert np.array_equal(got.view(np.uint64), golden["expw_y"].view(np.uint64))
    # domain contract (kernels.hpp:19-20): <= -708 -> 0, >= 710 -> inf
    assert oracle.exp_w([-708.0])[0] == 0.0
    assert np.isinf(oracle.exp_w([710.0])[0])
    assert np.isnan(oracle.exp_w([np.nan])[0])


def test_exp_w_accuracy(oracle):
    x = np.linspace(-700, 700, 20001)
    rel = np.abs(oracle.exp_w(x) / np.exp(x) - 1)
    assert rel.max() < 4 * 2.3e-16  # test_kernels.cpp:60-75 (<= 4 ulp)


@pytest.mark.parametrize("name", list(TABLES))
@pytest.mark.parametrize("rs", [0, 1, 2, 3])
def test_table_resampling_matches_golden(oracle, golden, name, rs):
    lw, n_out, seed = table(name)
    r = oracle.resample_table(rs, lw, n_out, (seed, 3, 11), mh_steps=8, bound=float(np.max(lw)))
    assert np.array_equal(r["left"], golden[f"table_{name}_{rs}_left"])
    assert np.array_equal(r["right"], golden[f"table_{name}_{rs}_right"])
    g = golden[f"table_{name}_{rs}_lmw"]
    if np.isnan(g):
        assert r["log_mean_weight"] is None
    else:
        assert r["log_mean_weight"] == g
    assert r["weight_evals"] == golden[f"table_{name}_{rs}_evals"]


def test_dead_table_raises(oracle):
    lw = np.full((5, 5), -np.inf)
    with pytest.raises(RuntimeError, match="all pair weights are zero"):
        oracle.resample_table(0, lw, 10, (1, 0, 0))
    with pytest.raises(ValueError, match="finite log_upper_bound"):
        oracle.resample_table(3, np.zeros((3, 3)), 3, (1, 0, 0))


def test_mh_zero_steps_identity(oracle):
    r = oracle.resample_table(2, np.zeros((3, 3)), 9, (3, 1, 1), mh_steps=0)
    assert list(r["left"]) == [m % 3 for m in range(9)]
    assert r["weight_evals"] == 0 and r["biased"] and r["log_mean_weight"] is None


@pytest.mark.parametrize("T", [0, 1, 2, 5, 6, 30, 1023, 1024])
def test_schedule_depth_and_pairs(oracle, T):
    # test_smoother.cpp:195-227: depth = ceil(log2(T+1)), exactly T pairs
    levels, pairs = oracle.schedule(T)
    assert levels == (int(np.ceil(np.log2(T + 1))) if T > 0 else 0)
    assert len(pairs) == T
    for lv, node, la, lb, rb in pairs:
        s = 1 << (lv - 1)
        assert la == 2 * node * s and lb == (2 * node + 1) * s - 1
        assert rb == min((2 * node + 2) * s - 1, T)


@pytest.mark.parametrize("name", list(CASES))
def test_smoother_matches_golden(oracle, golden, name):
    spec, m = golden_model(golden, name)
    for rs in spec["resamplers"]:
        r = oracle.smooth(m, spec["N"], rs, seed=spec["seed"], mh_steps=spec.get("mh_steps", 16))
        assert np.array_equal(r["leaves"], golden[f"case_{name}_states"])
        assert np.array_equal(r["pair_left"], golden[f"case_{name}_{rs}_left"])
        assert np.array_equal(r["pair_right"], golden[f"case_{name}_{rs}_right"])
        assert np.array_equal(r["paths"], golden[f"case_{name}_{rs}_paths"])
        g = golden[f"case_{name}_{rs}_lnc"]
        assert (r["log_norm_const"] is None) if np.isnan(g) else (r["log_norm_const"] == g)
        assert r["weight_evals"] == golden[f"case_{name}_{rs}_evals"]


@pytest.mark.parametrize("name", [n for n, s in CASES.items() if s.get("sweeps")])
def test_conditional_matches_golden(oracle, golden, name):
    spec, m = golden_model(golden, name)
    for sweep in spec["sweeps"]:
        ref = golden[f"case_{name}_cond{sweep}_ref"]
        r = oracle.conditional(m, ref, spec["N"], spec["seed"], sweep)
        assert np.array_equal(r["path"], golden[f"case_{name}_cond{sweep}_path"])
        assert r["log_norm_const"] == golden[f"case_{name}_cond{sweep}_lnc"]
        assert r["weight_evals"] == golden[f"case_{name}_cond{sweep}_evals"]


def test_conditional_rejects_ordered_resamplers(oracle, golden):
    spec, m = golden_model(golden, "ar1")
    ref = golden["case_ar1_cond1_ref"]
    for rs in (abi.SYSTEMATIC, abi.MH_LAZY):
        with pytest.raises(ValueError, match="exchangeable"):
            oracle.conditional(m, ref, 8, 1, 0, resampler=rs)


def test_oracle_matches_compiled_reference_fresh(oracle, reference):
    """Beyond the fixtures: fresh seeds against the compiled reference."""
    from paper_2202_02264_b200 import models
    m = models.lgssm_check(77)
    for seed in (1, 2):
        a = oracle.smooth(m, 29, 0, seed=seed)
        b = reference.run_smoother(m, 29, 0, seed=seed)
        assert np.array_equal(a["paths"], b["paths"])
        assert a["log_norm_const"] == b["log_norm_const"]


@pytest.mark.parametrize("kind,N,rs", [("cv", 40, abi.MULTINOMIAL), ("sv", 50, abi.MH_LAZY),
                                       ("crw", 64, abi.REJECTION_LAZY),
                                       ("lg", 9, abi.SYSTEMATIC)])
def test_reference_injected_runner(reference, kind, N, rs):
    """ref_run_injected (the full-size parity runner of
    tests/test_gpu_baseline_parity.py): replaying the reference's own leaves
    reproduces its level-by-level trace (pairs) and run_smoother's root, log Z,
    evals and bias flag."""
    from oracle.py import Oracle
    from paper_2202_02264_b200 import models
    m = {"cv": lambda: models.cv_tracking(63, smoother=Oracle().kalman_smooth),
         "sv": lambda: models.sv(77), "crw": lambda: models.constrained_rw(50),
         "lg": lambda: models.lgssm_check(6, smoother=Oracle().kalman_smooth)}[kind]()
    lv = reference.leaves(m, N, 7)
    X, W = reference.leaves_all(m, N, 7)
    assert np.array_equal(X, lv["states"]) and np.array_equal(W, lv["raw_logw"])
    assert np.array_equal(reference.leaf_weights(m, X), W)
    a = reference.trace_smoother(m, N, rs, seed=7, mh_steps=4)
    b = reference.run_injected(m, N, X, W, rs, seed=7, mh_steps=4, threads=3)
    c = reference.run_injected(m, N, X, None, rs, seed=7, mh_steps=4, want_pairs=False)
    s = reference.run_smoother(m, N, rs, seed=7, mh_steps=4)
    assert np.array_equal(a["pair_left"], b["pair_left"])
    assert np.array_equal(a["pair_right"], b["pair_right"])
    for r in (b, c):
        assert np.array_equal(r["paths"], s["paths"])
        assert r["log_norm_const"] == s["log_norm_const"]
        assert r["weight_evals"] == s["weight_evals"] and r["biased"] == s["biased"]


def test_oracle_kalman_matches_numpy():
    """or_kalman_smooth (the reference arm's RTS, kalman.cpp:78-138) against
    the independent numpy restatement."""
    from oracle.py import Oracle
    from paper_2202_02264_b200 import models
    from tests.test_abi import numpy_rts
    O = Oracle()
    for m in (models.cv_tracking(200, smoother=O.kalman_smooth),
              models.lgssm_check(100, smoother=O.kalman_smooth)):
        a, P, ll = O.kalman_smooth(m)
        b, Q = numpy_rts(m)
        assert np.allclose(a, b, rtol=1e-10, atol=1e-10) and np.allclose(P, Q, rtol=1e-10,
                                                                           atol=1e-12)
        assert np.isfinite(ll)


def test_gamma_draw_pinned_to_the_reference(oracle, reference):
    """gamma_draw (pgibbs.cpp:80-102) compiled from the reference's own source
    (oracle/Makefile extracts the function; pgibbs.cpp as a whole needs Eigen)
    against the oracle's restatement: bitwise over shapes below and above 1,
    several rates and streams (both use glibc pow/log/sqrt)."""
    for shape in (0.05, 0.3, 0.999, 1.0, 1.7, 3.0, 12.5, 2049.0):
        for rate in (0.01, 1.0, 37.0):
            for node in range(6):
                key = (99 + node, 0, node, abi.ROLE_GIBBS_PARAM)
                a = oracle.L.or_gamma_draw(shape, rate, *key)
                b = reference.gamma_draw(shape, rate, key)
                assert a == b, (shape, rate, node)
    with pytest.raises(ValueError):
        reference.gamma_draw(0.0, 1.0, (1, 0, 0, abi.ROLE_GIBBS_PARAM))


def test_sv_param_update_oracle_equals_reference_gamma(oracle, reference):
    """The SV parameter kernel restated in C (or_sv_param_update) equals the
    same kernel on the reference's RngStream + gamma_draw, bit for bit."""
    rng = np.random.default_rng(3)
    prior = abi.SvPrior(-1.0, 1.0, 2.0, 0.2, 0.05)
    for T in (0, 7, 511):
        for seed in (1, 77, 1234):
            x = -1.0 + 0.4 * rng.standard_normal(T + 1)
            th = np.array([-1.0, 0.9, 0.1]) + 0.01 * rng.standard_normal(3)
            a, acc_a = oracle.sv_param_update(x, th, prior, seed, 3)
            b, acc_b = reference.sv_param_update(x, th, prior, seed, 3)
            assert np.array_equal(a, b) and acc_a == acc_b
