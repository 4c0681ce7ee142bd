"""TEST INFRASTRUCTURE: golden config hashes of the experiment harness.

Builds tests/golden/hash_probe.cpp against the JSON library the reference's
harness links (nlohmann/json, present in this image under cudnn_frontend's
third-party tree) and records, for a few harness config files, the hash the
reference's config_hash (experiment.cpp:240-303) gives. The CPU test
tests/test_harness.py checks that dsmc_cli writes the same config_hash.

    python tests/golden/make_hash_golden.py
"""
import glob
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "hash_golden.json")

DEFAULT = dict(experiment="cox", T=32, N=256, replicates=10, methods=[], resampler="multinomial",
               mh_steps=16, seed=1, data_seed=90210, proposal_inflation=1.0, sweeps=1000,
               cox=dict(mu=0.0, rho=0.9, sigma2=0.25, **{"lambda": 1.0}), rw=dict(sigma=0.5),
               theta=dict(tau0=0.15, tau1=0.10, tau2=0.10, q2=0.05, r2=0.05),
               lgssm=dict(coef=0.9, shift=0.0, trans_var=0.25, init_mean=0.0, init_var=1.0,
                          obs_var=0.25),
               gibbs=dict(prec_x_shape=2.0, prec_x_rate=1.0, prec_y_shape=2.0, prec_y_rate=1.0,
                          tau0_sd=1.0, tau1_sd=1.0, tau2_sd=1.0, rwm_step_tau=0.05,
                          rwm_step_x0=0.1, ieks_cold_iterations=25))

# config-file overlays (harness JSON keys)
CASES = [
    {},
    dict(experiment="constrained-rw", T=63, N=512, replicates=3),
    dict(experiment="lgssm-check", T=31, N=128, methods=["dsmc", "dsmc-mh"], mh_steps=8,
         seed=123456789012345678, proposal_inflation=1e-05,
         lgssm=dict(coef=-0.25, shift=3.0, trans_var=1e20, obs_var=12345.678)),
    dict(experiment="theta-logistic", T=100, N=64, resampler="systematic", sweeps=50,
         theta=dict(tau0=0.123456789, tau1=1e-7, tau2=2.5e-3),
         gibbs=dict(rwm_step_tau=0.0, ieks_cold_iterations=3, prec_x_rate=1234567890123456.0)),
]


def merged(over):
    c = json.loads(json.dumps(DEFAULT))
    for k, v in over.items():
        if isinstance(v, dict):
            c[k].update(v)
        else:
            c[k] = v
    return c


def probe_line(c):
    methods = c["methods"] or (["dsmc", "dsmc-rs", "ffbs"] if c["experiment"] == "constrained-rw"
                               else ["dsmc", "ffbs"])
    x, th, lg, g = c["cox"], c["theta"], c["lgssm"], c["gibbs"]
    vals = [c["experiment"], c["T"], c["N"], c["replicates"], ",".join(methods), c["resampler"],
            c["mh_steps"], c["seed"], c["data_seed"], repr(c["proposal_inflation"]), c["sweeps"],
            x["mu"], x["rho"], x["sigma2"], x["lambda"], c["rw"]["sigma"], th["tau0"], th["tau1"],
            th["tau2"], th["q2"], th["r2"], lg["coef"], lg["shift"], lg["trans_var"],
            lg["init_mean"], lg["init_var"], lg["obs_var"], g["prec_x_shape"], g["prec_x_rate"],
            g["prec_y_shape"], g["prec_y_rate"], g["tau0_sd"], g["tau1_sd"], g["tau2_sd"],
            g["rwm_step_tau"], g["rwm_step_x0"], g["ieks_cold_iterations"]]
    return " ".join(repr(v) if isinstance(v, float) else str(v) for v in vals)


def main():
    inc = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                 "cudnn_frontend", "thirdparty"))[0]
    exe = "/tmp/hash_probe"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + inc, os.path.join(HERE, "hash_probe.cpp"),
                    "-o", exe], check=True)
    cases = []
    for over in CASES:
        c = merged(over)
        r = subprocess.run([exe], input=probe_line(c) + "\n", capture_output=True, text=True,
                           check=True).stdout.split()
        cases.append(dict(config=over, hash=r[0], dump=r[1]))
    json.dump(dict(cases=cases), open(OUT, "w"), indent=1)
    print("wrote", OUT, [c["hash"] for c in cases])


if __name__ == "__main__":
    main()
