"""The experiment harness (paper_2202_02264_b200/dsmc_cli):
the reference's CLI subcommands, JSON config overlay, config hash and
fixed-schema result CSV (tools/dsmc_cli.cpp, tools/experiment.cpp).

CPU tests cover argument/config handling, the CSV schema and the config hash
(pinned by tests/golden/hash_golden.json, generated with the JSON library the
reference links); the host data simulators and RNG run in test_host's cpu_
cases. GPU tests run every subcommand and pin FP64 rows to the compiled
reference (tests/golden/harness_golden.json): same seeds, levels and
weight_evals, estimates and log Z to 1e-12."""
import csv
import io
import json
import math
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2202_02264_b200", "dsmc_cli")
HOSTBIN = os.path.join(ROOT, "tests", "cpp", "test_host")
GOLD = os.path.join(ROOT, "tests", "golden")
HEADER = ("experiment,T,N,method,replicate,estimate,wall_time_ms,levels,weight_evals,"
          "log_norm_const,seed,config_hash,error")


def run(args, cwd, timeout=600):
    return subprocess.run([CLI] + args, capture_output=True, text=True, cwd=cwd, timeout=timeout)


def read_rows(path):
    text = open(path).read()
    assert text.splitlines()[0] == HEADER
    return list(csv.DictReader(io.StringIO(text)))


def test_cli_is_built():
    assert os.path.exists(CLI), "make -C paper_2202_02264_b200/csrc"


def test_host_only_cases_pass():
    r = subprocess.run([HOSTBIN, "cpu_"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failing cases" in r.stdout


@pytest.mark.parametrize("args,code,msg", [
    ([], 2, "usage"),
    (["frobnicate"], 2, "unknown subcommand"),
    (["smooth", "--bogus", "1"], 2, "not expected: --bogus"),
    (["smooth", "--sweeps", "3"], 2, "not expected: --sweeps"),
    (["pgibbs", "--methods", "dsmc"], 2, "not expected: --methods"),
    (["smooth", "--experiment", "foo"], 2, "unknown experiment: foo"),
    (["smooth", "--N", "1"], 2, "N must be at least 2"),
    (["smooth", "--T", "0"], 2, "T must be at least 1"),
    (["smooth", "--methods", "dsmc,pf"], 2, "unknown method: pf"),
    (["smooth", "--resampler", "stratified"], 2, "unknown resampler: stratified"),
    (["smooth", "--resampler", "mh-lazy"], 2, "stitches with a dense scheme"),
    (["smooth", "--inflation", "0"], 2, "proposal inflation must be positive"),
    (["pgibbs", "--experiment", "cox"], 2, "pgibbs runs the theta-logistic experiment only"),
    (["check-oracle", "--replicates", "3"], 2, "at least 4 replicates"),
    (["bench", "--T-list", "8,0"], 2, "--T-list entries must be at least 1"),
    (["smooth", "--T", "x"], 2, "not an integer"),
])
def test_usage_and_validation_errors(tmp_path, args, code, msg):
    r = run(args, tmp_path)
    assert r.returncode == code
    assert msg in r.stderr + r.stdout


def test_json_config_rejects_unknown_and_malformed(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"experiment": "cox", "Tee": 3}))
    r = run(["smooth", "--config", str(p)], tmp_path)
    assert r.returncode == 2 and "unknown config key 'Tee' in the top-level object" in r.stderr
    p.write_text(json.dumps({"cox": {"mu": 0.0, "nu": 1.0}}))
    r = run(["smooth", "--config", str(p)], tmp_path)
    assert r.returncode == 2 and "unknown config key 'nu' in \"cox\"" in r.stderr
    p.write_text("{\"T\": 3,")
    r = run(["smooth", "--config", str(p)], tmp_path)
    assert r.returncode == 2 and "malformed JSON" in r.stderr
    r = run(["smooth", "--config", str(tmp_path / "missing.json")], tmp_path)
    assert r.returncode == 2 and "cannot open config file" in r.stderr


def test_config_hash_matches_the_reference_json_dump(tmp_path):
    g = json.load(open(os.path.join(GOLD, "hash_golden.json")))
    for case in g["cases"]:
        p = tmp_path / "c.json"
        p.write_text(json.dumps(case["config"]))
        out = tmp_path / "o.csv"
        run(["smooth", "--config", str(p), "--out", str(out)], tmp_path)
        rows = read_rows(out)
        assert rows and all(r["config_hash"] == case["hash"] for r in rows), case


def test_flags_override_config_and_rows_follow_the_schema(tmp_path):
    """Without a GPU every row records the failure in its error column (no CPU
    fallback); the schema, the method-major row order, the derived seeds and
    the flag-over-config precedence still hold."""
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"experiment": "lgssm-check", "T": 7, "N": 16, "replicates": 2,
                             "methods": ["ffbs", "dsmc"], "seed": 5}))
    out = tmp_path / "o.csv"
    r = run(["smooth", "--config", str(p), "--T", "9", "--out", str(out), "--stable-timing"],
            tmp_path)
    rows = read_rows(out)
    assert [(x["method"], x["replicate"]) for x in rows] == [
        ("ffbs", "0"), ("ffbs", "1"), ("dsmc", "0"), ("dsmc", "1")]
    assert all(x["T"] == "9" and x["N"] == "16" for x in rows)
    # derive_seed: base + ((method_id + 1) << 32) + replicate
    assert [int(x["seed"]) for x in rows] == [5 + (4 << 32), 6 + (4 << 32), 5 + (1 << 32),
                                              6 + (1 << 32)]
    if r.returncode != 0:  # no device here: loud failure, never a CPU answer
        assert all(x["error"] and x["estimate"] == "" for x in rows)
        assert all(x["wall_time_ms"] == "0" for x in rows)


# ----------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "harness_golden.json")))["cases"],
                         ids=lambda c: c["experiment"])
def test_fp64_rows_equal_the_reference(tmp_path, case):
    """dsmc_cli smooth --precision fp64 reproduces the compiled reference's
    rows (same simulated data, same seeds): levels and weight_evals exactly,
    estimate and log Z to 1e-12 relative. The device's FP64 log/sin/cos in the
    leaf draws differ from glibc's by <= 1 ulp (test_gpu_parity.py pins the
    paths bitwise with injected leaves), so the states carry ulp-level noise;
    any different ancestor draw would move the estimate by ~1e-3."""
    out = tmp_path / "o.csv"
    r = run(["smooth", "--experiment", case["experiment"], "--T", str(case["T"]), "--N",
             str(case["N"]), "--replicates", str(len(case["rows"])), "--methods", "dsmc",
             "--precision", "fp64", "--stable-timing", "--out", str(out)], tmp_path)
    assert r.returncode == 0, r.stderr
    rows = read_rows(out)
    for got, want in zip(rows, case["rows"]):
        assert got["error"] == ""
        assert int(got["seed"]) == want["seed"]
        assert float(got["estimate"]) == pytest.approx(want["estimate"], rel=1e-12, abs=1e-13)
        assert float(got["log_norm_const"]) == pytest.approx(want["log_norm_const"], rel=1e-12)
        assert int(got["levels"]) == want["levels"]
        assert int(got["weight_evals"]) == want["weight_evals"]


@pytest.mark.gpu
def test_smooth_is_byte_stable_and_every_method_runs(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    args = ["smooth", "--experiment", "constrained-rw", "--T", "63", "--N", "256",
            "--replicates", "2", "--methods", "dsmc,dsmc-rs,dsmc-mh,ffbs", "--stable-timing"]
    r1 = run(args + ["--out", str(a)], tmp_path)
    r2 = run(args + ["--out", str(b)], tmp_path)
    assert r1.returncode == 0 and r2.returncode == 0, r1.stderr
    assert a.read_bytes() == b.read_bytes()
    rows = read_rows(a)
    assert len(rows) == 8 and all(x["error"] == "" for x in rows)
    for x in rows:
        assert float(x["estimate"]) > 0  # log(0.5) + sum of squared steps / sigma^3
        if x["method"] in ("dsmc", "ffbs"):
            assert x["log_norm_const"] != ""
        if x["method"] == "dsmc-mh":  # lazy: no normalising constant
            assert x["log_norm_const"] == ""
    assert "4/" not in r1.stdout or "replicates ok" in r1.stdout


@pytest.mark.gpu
def test_smooth_cox_and_theta_logistic(tmp_path):
    for exp in ("cox", "theta-logistic"):
        out = tmp_path / f"{exp}.csv"
        r = run(["smooth", "--experiment", exp, "--T", "127", "--N", "512", "--replicates", "3",
                 "--out", str(out)], tmp_path)
        assert r.returncode == 0, r.stderr
        rows = read_rows(out)
        assert len(rows) == 6 and all(x["error"] == "" for x in rows)
        est = {m: [float(x["estimate"]) for x in rows if x["method"] == m] for m in ("dsmc", "ffbs")}
        assert all(math.isfinite(v) for vs in est.values() for v in vs)
        if exp == "theta-logistic":
            # both smoothers estimate E[x_T | y]; the Cox score functional is
            # too noisy at this size for a 3-replicate comparison
            md, mf = sum(est["dsmc"]) / 3, sum(est["ffbs"]) / 3
            assert abs(md - mf) < 0.25 * (abs(md) + abs(mf)) + 0.5, (exp, est)


@pytest.mark.gpu
def test_threads_give_the_same_rows(tmp_path):
    """--threads runs replicates on several host threads (one engine context
    each): the rows (seeded per replicate) are the same as a serial run."""
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    args = ["smooth", "--experiment", "lgssm-check", "--T", "63", "--N", "128",
            "--replicates", "6", "--stable-timing"]
    r1 = run(args + ["--out", str(a)], tmp_path)
    r2 = run(args + ["--threads", "3", "--out", str(b)], tmp_path)
    assert r1.returncode == 0 and r2.returncode == 0, r2.stderr
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_check_oracle_passes(tmp_path):
    r = run(["check-oracle", "--T", "63", "--N", "512", "--replicates", "8"], tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 3 and "[FAIL]" not in r.stdout


@pytest.mark.gpu
def test_pgibbs_rows_and_trace(tmp_path):
    out, trace = tmp_path / "p.csv", tmp_path / "t.csv"
    r = run(["pgibbs", "--T", "60", "--N", "64", "--replicates", "2", "--sweeps", "6",
             "--trace", str(trace), "--out", str(out)], tmp_path)
    assert r.returncode == 0, r.stderr
    assert "synthetic theta-logistic data" in r.stderr
    rows = read_rows(out)
    assert len(rows) == 2 and all(x["method"] == "dsmc" and x["error"] == "" for x in rows)
    for x in rows:
        assert 0.0 < float(x["estimate"]) <= 1.0  # mean per-time update rate
        assert int(x["levels"]) == 6 and int(x["weight_evals"]) > 0
    t = trace.read_text().splitlines()
    assert t[0] == "chain,sweep,tau0,tau1,tau2,q2,r2" and len(t) == 1 + 2 * 6
    assert all(float(v) > 0 for line in t[1:] for v in line.split(",")[5:7])


@pytest.mark.gpu
def test_bench_grid(tmp_path):
    out = tmp_path / "b.csv"
    r = run(["bench", "--experiment", "lgssm-check", "--T-list", "15,31", "--N-list", "32,64",
             "--replicates", "1", "--out", str(out)], tmp_path)
    assert r.returncode == 0, r.stderr
    rows = read_rows(out)
    assert [(x["T"], x["N"], x["method"]) for x in rows] == [
        (t, n, m) for t in ("15", "31") for n in ("32", "64") for m in ("dsmc", "ffbs")]
