"""TEST INFRASTRUCTURE: a CPU backend for the time-sharded protocol
(paper_2202_02264_b200/sharded.py), so the multi-rank host logic (windows,
global stream keys, boundary exchange, index remaps, cross-level composition)
is exercised over gloo on CPU. Same five stages as GpuBackend, computed with
numpy and the oracle's table resampler (resampling.cpp restated) on a d=1
linear-Gaussian model. Not the product (that is GpuBackend)."""
import math

import numpy as np
import torch

from paper_2202_02264_b200 import abi

L2P = math.log(2 * math.pi)


def lnp(x, m, v):
    return -0.5 * (L2P + np.log(v)) - (x - m) ** 2 / (2 * v)


class CpuBackend:
    comm_device = torch.device("cpu")

    def __init__(self, model, N, seed, oracle, resampler=abi.MULTINOMIAL, mh_steps=4):
        A = model.arrays
        g = lambda k: np.asarray(A[k], float).ravel()
        self.F, self.b, self.Q, self.H, self.R = (float(g(k)[0]) for k in "F b Q H R".split())
        self.y, self.pm, self.pv = g("y"), g("prop_mean"), g("prop_cov")
        self.m0, self.P0 = float(g("m0")[0]), float(g("P0")[0])
        self.N, self.seed, self.O = N, seed, oracle
        self.resampler, self.mh_steps = resampler, mh_steps
        self.len = 0

    def empty_states(self):
        return torch.zeros((self.N, 4), dtype=torch.float32)

    def empty_col(self):
        return torch.zeros(self.N, dtype=torch.float32)

    def empty_idx(self):
        return torch.zeros(self.N, dtype=torch.int32)

    def sync(self):
        pass

    # leaves keyed by the GLOBAL time
    def _leaf(self, t):
        z = np.random.default_rng([self.seed, t]).standard_normal(self.N)
        x = self.pm[t] + np.sqrt(self.pv[t]) * z
        col = lnp(self.y[t], self.H * x, self.R) - lnp(x, self.pm[t], self.pv[t])
        if t >= 1:
            col = col - 0.5 * (L2P + np.log(self.Q))
        lw = None
        if t == 0:
            raw = lnp(self.y[0], self.H * x, self.R) + lnp(x, self.m0, self.P0) - lnp(x, self.pm[0], self.pv[0])
            m = raw.max()
            lse = m + np.log(np.exp(raw - m).sum())
            lw = raw - lse
            lnc = lse - np.log(self.N)
        else:
            lnc = 0.0
        return x.astype(np.float32), col.astype(np.float32), lw, lnc

    def _combine(self, xl, xr, colr, lwl, level, node, lnc_l, lnc_r):
        xl = xl.astype(np.float64)
        xr = xr.astype(np.float64)
        mu = self.F * xl + self.b
        table = colr.astype(np.float64)[None, :] - (xr[None, :] - mu[:, None]) ** 2 / (2 * self.Q)
        if lwl is not None:
            table = table + lwl[:, None]
        # rejection: the table max is a valid (exact) bound for this test model
        r = self.O.resample_table(self.resampler, table, self.N, (self.seed, level, node),
                                  mh_steps=self.mh_steps, bound=float(np.max(table)))
        shift = (-np.log(self.N) if lwl is None else 0.0) - np.log(self.N)
        lmw = r["log_mean_weight"]
        return r["left"].astype(np.int64), r["right"].astype(np.int64), \
            (lnc_l + lnc_r + lmw + shift) if lmw is not None else float("nan")

    def window_run(self, t0, length):
        self.t0, self.len = t0, length
        self.X, self.C, lw0, self.LNC = {}, {}, None, {}
        for t in range(length):
            x, c, lw, lnc = self._leaf(t0 + t)
            self.X[t], self.C[t], self.LNC[t] = x, c, lnc
            if lw is not None:
                lw0 = lw
        # blocks: (a, b) local, first/last maps, lnc
        blocks = [dict(a=t, b=t, first=np.arange(self.N), last=np.arange(self.N),
                       lnc=self.LNC[t]) for t in range(length)]
        self.pairs = {}
        level = 0
        while len(blocks) > 1:
            level += 1
            nxt = []
            for k in range(len(blocks) // 2):
                Lb, Rb = blocks[2 * k], blocks[2 * k + 1]
                c = Rb["a"]
                xl = self.X[c - 1][Lb["last"]]
                xr = self.X[c][Rb["first"]]
                colr = self.C[c][Rb["first"]]
                lwl = lw0 if (Lb["a"] == Lb["b"] and t0 + Lb["a"] == 0) else None
                l, r, lnc = self._combine(xl, xr, colr, lwl, level, (t0 >> level) + k,
                                          Lb["lnc"], Rb["lnc"])
                self.pairs[(level, k)] = (l, r)
                nxt.append(dict(a=Lb["a"], b=Rb["b"], first=Lb["first"][l], last=Rb["last"][r],
                                lnc=lnc))
            blocks = nxt
        self.levels = level
        self.root = blocks[0]

    def root_lnc(self, out):
        out.fill_(float(self.root["lnc"]))

    def boundary(self, side):
        x = self.empty_states()
        if side == 0:
            x[:, 0] = torch.from_numpy(self.X[0][self.root["first"]])
            col = torch.from_numpy(self.C[0][self.root["first"]].copy())
            return x, col
        x[:, 0] = torch.from_numpy(self.X[self.len - 1][self.root["last"]])
        return x, None

    def cross(self, cut, level, node, xl, xr, colr, lnc_l, lnc_r, lnc_out):
        l, r, lnc = self._combine(xl[:, 0].numpy(), xr[:, 0].numpy(), colr.numpy(), None, level,
                                  node, float(lnc_l[0]), float(lnc_r[0]))
        lnc_out.fill_(lnc)
        return torch.from_numpy(l.astype(np.int32)), torch.from_numpy(r.astype(np.int32))

    def remap(self, side, idx):
        key = "first" if side == 0 else "last"
        self.root[key] = self.root[key][idx.numpy().astype(np.int64)]

    def finish(self, root_map):
        maps = {(self.levels, 0): np.asarray(root_map.cpu() if torch.is_tensor(root_map)
                                             else root_map, np.int64)}
        for level in range(self.levels, 0, -1):
            for k in range(self.len >> level):
                M = maps[(level, k)]
                l, r = self.pairs[(level, k)]
                maps[(level - 1, 2 * k)] = l[M]
                maps[(level - 1, 2 * k + 1)] = r[M]
        mean = torch.zeros((self.len, 1), dtype=torch.float64)
        cov = torch.zeros((self.len, 1, 1), dtype=torch.float64)
        for t in range(self.len):
            x = self.X[t][maps[(0, t)]].astype(np.float64)
            mean[t, 0] = x.mean()
            cov[t, 0, 0] = x.var()
        return mean, cov
