"""Generate the golden fixtures in tests/golden/ from the COMPILED REFERENCE.

Run here (the reference exists only in this container):
    make -C oracle all && python tests/golden/make_golden.py

Every array comes from /root/reference's own code (oracle/_ref/libdsmc_ref.so:
rng.cpp, kernels/*.cpp, resampling.cpp, smoother.cpp, conditional.cpp compiled
unmodified; models restated in oracle/ref_models.cpp). The reference ships no
golden vectors for ancestor indices, so these are its outputs on
seeded inputs; the Philox known-answer vectors are the reference's own
(test_rng.cpp:32-47).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.py import Reference  # noqa: E402
from paper_2202_02264_b200 import abi, models  # noqa: E402
from tests.cases import CASES, TABLES, model_arrays, model_for, table  # noqa: E402


def main():
    R = Reference()
    out = {}
    # Philox KAT (test_rng.cpp:32-47) + stream draws of each kind
    out["kat_z"] = R.philox([0, 0, 0, 0], [0, 0])
    out["kat_w"] = R.philox([0xDEADBEEF, 1, 2, 3], [0x9E3779B97F4A7C15, 0x243F6A8885A308D3])
    for kind in ("u64", "uniform", "uniform_pos", "normal"):
        out[f"stream_{kind}"] = R.stream((42, 3, 17, abi.ROLE_PAIR_RESAMPLE), kind, 257, substream=5)
    # exp_w over its domain edges and a dense grid (exp_poly.hpp:39-51)
    xs = np.r_[np.linspace(-720, 720, 4001), -708.0, -707.9999, 709.9, 710.0, 711.0,
               -np.inf, np.inf, 0.0, -0.0, 1e-300, -1e-300]
    out["expw_x"] = xs
    out["expw_y"] = np.array([R.L.ref_exp_w(float(v)) for v in xs])
    # table resampling (resampling.cpp:181-324)
    for name in TABLES:
        lw, n_out, seed = table(name)
        for rs in range(4):
            r = R.resample_table(rs, lw, n_out, (seed, 3, 11), mh_steps=8,
                                 bound=float(np.max(lw)))
            out[f"table_{name}_{rs}_left"] = r["left"]
            out[f"table_{name}_{rs}_right"] = r["right"]
            out[f"table_{name}_{rs}_lmw"] = np.float64(np.nan if r["log_mean_weight"] is None
                                                       else r["log_mean_weight"])
            out[f"table_{name}_{rs}_evals"] = np.uint64(r["weight_evals"])
    # smoother traces (run_smoother through make_leaf / make_pair_source /
    # resample_pairs / combine_blocks)
    for name, spec in CASES.items():
        m = model_for(spec)
        for k, v in model_arrays(m).items():
            out[f"case_{name}_model_{k}"] = v
        N, seed = spec["N"], spec["seed"]
        lv = R.leaves(m, N, seed)
        out[f"case_{name}_states"] = lv["states"]
        out[f"case_{name}_raw_logw"] = lv["raw_logw"]
        for rs in spec["resamplers"]:
            tr = R.trace_smoother(m, N, rs, seed=seed, mh_steps=spec.get("mh_steps", 16))
            full = R.run_smoother(m, N, rs, seed=seed, mh_steps=spec.get("mh_steps", 16))
            assert np.array_equal(tr["paths"], full["paths"])
            out[f"case_{name}_{rs}_left"] = tr["pair_left"]
            out[f"case_{name}_{rs}_right"] = tr["pair_right"]
            out[f"case_{name}_{rs}_lmw"] = tr["log_mean_weight"]
            out[f"case_{name}_{rs}_paths"] = tr["paths"]
            out[f"case_{name}_{rs}_lnc"] = np.float64(np.nan if full["log_norm_const"] is None
                                                      else full["log_norm_const"])
            out[f"case_{name}_{rs}_evals"] = np.uint64(full["weight_evals"])
        for sweep in spec.get("sweeps", []):
            ref_path = lv["states"][:, 0, :]  # any fixed path on the support
            c = R.conditional(m, ref_path, N, seed, sweep)
            out[f"case_{name}_cond{sweep}_states"] = R.conditional_leaves(m, ref_path, N, seed, sweep)
            out[f"case_{name}_cond{sweep}_ref"] = ref_path
            out[f"case_{name}_cond{sweep}_path"] = c["path"]
            out[f"case_{name}_cond{sweep}_lnc"] = np.float64(c["log_norm_const"])
            out[f"case_{name}_cond{sweep}_evals"] = np.uint64(c["weight_evals"])
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(out)} arrays")


if __name__ == "__main__":
    main()
