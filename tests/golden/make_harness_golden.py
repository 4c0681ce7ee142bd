"""TEST INFRASTRUCTURE: golden rows for the experiment harness (dsmc_cli).

Run here (where oracle/_ref was compiled from /root/reference); the output
tests/golden/harness_golden.json travels to the GPU box. For each case it
records the reference's answer for one `dsmc_cli smooth --methods dsmc
--precision fp64` row:

  * the data set, simulated with the reference's own Philox block function
    (oracle/_ref ref_philox) driven by a restatement of RngStream
    (rng.cpp:45-93) and of simulate_cox / simulate_lgssm
    (models.cpp:230-252, kalman.cpp:157-175);
  * the reference smoother's root population (oracle/_ref ref_run_smoother,
    FP64) on that data, reduced to the harness estimate
    (experiment.cpp:470-482 block_functional_mean with cox_score /
    rw_score / path[T], models.cpp:218-228,340-347) and log Z;
  * seeds derive_seed(seed, 0, replicate) (experiment.cpp:39-45).

    python tests/golden/make_harness_golden.py
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.py import Reference  # noqa: E402
from paper_2202_02264_b200 import abi, models  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "harness_golden.json")
M64 = (1 << 64) - 1


class Stream:
    """RngStream restated over the reference's philox4x64_10."""

    def __init__(self, ref, seed, level, node, role, sub=0):
        self.ref = ref
        self.ctr = [0, node, ((level << 16) | role) & M64, sub]
        self.key = [seed, 0x243F6A8885A308D3]
        self.buf, self.pos, self.cached = None, 4, None

    def u64(self):
        if self.pos == 4:
            self.buf = [int(v) for v in self.ref.philox(self.ctr, self.key)]
            self.ctr[0] += 1
            self.pos = 0
        v = self.buf[self.pos]
        self.pos += 1
        return v

    def uniform(self):
        return float(self.u64() >> 11) * 2.0 ** -53

    def uniform_pos(self):
        return (float(self.u64() >> 12) + 0.5) * 2.0 ** -52

    def normal(self):
        if self.cached is not None:
            v, self.cached = self.cached, None
            return v
        u1 = self.uniform_pos()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 2.0 * math.pi * u2
        self.cached = r * math.sin(th)
        return r * math.cos(th)


def simulate_cox(ref, T, seed, mu=0.0, rho=0.9, sigma2=0.25, lam=1.0):
    a, c = rho * lam, mu * (1.0 - rho)
    st = Stream(ref, seed, 0, 0, 5)
    xs = [c / (1.0 - a) + math.sqrt(sigma2 / (1.0 - a * a)) * st.normal()]
    for _ in range(T):
        xs.append(c + a * xs[-1] + math.sqrt(sigma2) * st.normal())
    ys = []
    for x in xs:
        rate, total = math.exp(x), 0
        while rate > 0.0:
            chunk = min(rate, 30.0)
            rate -= chunk
            limit, prod, k = math.exp(-chunk), 1.0, 0
            while True:
                k += 1
                prod *= st.uniform_pos()
                if not prod > limit:
                    break
            total += k - 1
        ys.append(float(total))
    return ys


def simulate_lgssm_check(ref, T, seed, coef=0.9, shift=0.0, q=0.25, m0=0.0, p0=1.0, r=0.25):
    st = Stream(ref, seed, 0, 0, 5)
    xs = [m0 + math.sqrt(p0) * st.normal()]
    for _ in range(T):
        xs.append(coef * xs[-1] + shift + math.sqrt(q) * st.normal())
    return [1.0 * x + math.sqrt(r) * st.normal() for x in xs]


def cox_score(path, T, mu=0.0, rho=0.9, s2=0.25):
    d0 = path[0] - mu
    acc = -(T + 1) / (2.0 * s2)
    acc += (1.0 - rho * rho) / (2.0 * s2 * s2) * d0 * d0
    for s in range(1, T + 1):
        e = path[s] - mu - rho * (path[s - 1] - mu)
        acc += e * e / (2.0 * s2 * s2)
    return acc


def rw_score(path, T, sigma):
    acc = 0.0
    for t in range(1, T + 1):
        d = path[t] - path[t - 1]
        acc += d * d
    return math.log(sigma) + acc / (sigma * sigma * sigma)


def derive_seed(base, method, rep):
    return (base + ((method + 1) << 32) + rep) & M64


def rows(ref, model, f, T, N, reps, seed=1):
    out = []
    for rep in range(reps):
        s = derive_seed(seed, 0, rep)
        r = ref.run_smoother(model, N, abi.MULTINOMIAL, seed=s)
        paths = r["paths"][:, :, 0]  # (K, N)
        lw = -math.log(N)
        acc = 0.0
        for i in range(N):
            acc += math.exp(lw) * f([float(v) for v in paths[:, i]])
        out.append(dict(replicate=rep, seed=s, estimate=acc, log_norm_const=r["log_norm_const"],
                        levels=r["levels"], weight_evals=r["weight_evals"]))
    return out


def main():
    ref = Reference()
    cases = []
    T, N = 15, 64
    ys = simulate_cox(ref, T, 90210)
    m = models.cox(T, ys=np.array(ys))
    cases.append(dict(experiment="cox", T=T, N=N, ys=ys,
                      rows=rows(ref, m, lambda p: cox_score(p, T), T, N, 2)))
    T, N = 31, 128
    ys = simulate_lgssm_check(ref, T, 90210)
    m = models.lgssm_check(T, ys=np.array(ys))
    cases.append(dict(experiment="lgssm-check", T=T, N=N, ys=ys,
                      rows=rows(ref, m, lambda p: p[T], T, N, 2)))
    T, N, sigma = 20, 64, 0.5
    m = models.constrained_rw(T, sigma)
    cases.append(dict(experiment="constrained-rw", T=T, N=N, ys=[],
                      rows=rows(ref, m, lambda p: rw_score(p, T, sigma), T, N, 2)))
    with open(OUT, "w") as fh:
        json.dump(dict(cases=cases), fh, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
