"""Time-sharded dSMC over several GPUs (the reference has no
distribution).

K = 2^k leaves, P ranks (P a power of two, K/P >= 2): rank g owns the window
[g K/P, (g+1) K/P) and runs its leaves and the log2(K/P) local levels with the
reference's GLOBAL stream keys ({seed, level, global node}), so the local
combines are exactly the ones a 1-GPU run performs. The top log2(P) levels
cross windows: for the combine at cut c (left block's last window gL, right
block's first window gR, left block's first window gA, right block's last
window gB):

  gR -> gL   R's first-leaf slab through R's first map (N states + N column
             terms), gathered on the device (dsmc_window_boundary)
  gL         runs the N x N combine with key {seed, level, node}
             (dsmc_cross_combine) -> (l, r), block log Z
  gL -> gA   l, so gA sets first := first[l]   (dsmc_window_remap)
  gL -> gB   r, so gB sets last  := last[r]

Block log Z values stay on the device and are all-reduced after each level
(a few doubles), the cross-level (l, r) once at the end; every rank then
composes its window's root map through the cross levels (device indexing)
and finishes its window locally (top-down composition + per-time moments).
No stage synchronises the host: the engine enqueues, NCCL P2P and the
reductions run on the engine stream, and device errors surface at the next
dsmc_sync. Exchanged bytes per cut: 20 N (slab) + 8 N (indices), latency
bound on NVLink. Any resampler works across windows (dense, MH-lazy,
rejection-lazy; log Z is NaN after a lazy level, as in the reference).

Transports: `TorchComm` (torch.distributed: NCCL on GPUs, gloo on CPU) and
in-process virtual ranks (several backends hosted by one process exchange
tensors directly). Backends: `GpuBackend` (the CUDA engine); tests add a CPU
backend implementing the same five stages.
"""
import contextlib
import math

import numpy as np
import torch

from . import abi


def _log2(x):
    v = int(round(math.log2(x)))
    if 1 << v != x:
        raise ValueError(f"{x} is not a power of two")
    return v


class GpuBackend:
    """One rank's CUDA engine context + uploaded model (use
    Engine.upload_window for a rank that only needs its window)."""

    def __init__(self, engine, handle, N, d, seed, resampler=abi.MULTINOMIAL, device=0,
                 mh_steps=16):
        self.e, self.h, self.N, self.d = engine, handle, N, d
        self.seed, self.resampler, self.mh_steps = seed, resampler, mh_steps
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(engine.stream_handle(), device=self.dev)
        self.len = 0

    # tensors of the exchange (torch's current stream = the engine stream)
    def empty_states(self):
        return torch.empty((self.N, 4), dtype=torch.float32, device=self.dev)

    def empty_col(self):
        return torch.empty(self.N, dtype=torch.float32, device=self.dev)

    def empty_idx(self):
        return torch.empty(self.N, dtype=torch.int32, device=self.dev)

    @property
    def comm_device(self):
        return self.dev

    def window_run(self, t0, length):
        self.len = length
        self.e.window_run(self.h, self.N, t0, length, self.seed, self.resampler, self.mh_steps)

    def root_lnc(self, out):
        """The window root's log Z into `out` (a 1-element device tensor)."""
        self.e.window_boundary(1, None, None, out.data_ptr())

    def boundary(self, side):
        x = self.empty_states()
        col = self.empty_col() if side == 0 else None
        self.e.window_boundary(side, x.data_ptr(), col.data_ptr() if col is not None else None)
        return x, col

    def cross(self, cut, level, node, xl, xr, colr, lnc_l, lnc_r, lnc_out):
        l, r = self.empty_idx(), self.empty_idx()
        self.e.cross_combine(self.h, self.N, self.seed, cut, level, node, xl.data_ptr(),
                             xr.data_ptr(), colr.data_ptr(), lnc_l.data_ptr(), lnc_r.data_ptr(),
                             l.data_ptr(), r.data_ptr(), lnc_out.data_ptr(), self.resampler,
                             self.mh_steps)
        return l, r

    def remap(self, side, idx):
        self.e.window_remap(side, idx.data_ptr())

    def finish(self, root_map):
        rm = root_map.to(device=self.dev, dtype=torch.int32).contiguous()
        mean = torch.empty((self.len, self.d), dtype=torch.float64, device=self.dev)
        cov = torch.empty((self.len, self.d, self.d), dtype=torch.float64, device=self.dev)
        self.e.window_finish(rm.data_ptr(), mean.data_ptr(), cov.data_ptr())
        return mean, cov

    def sync(self):
        self.e.sync()


class TorchComm:
    """torch.distributed transport (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        # gloo cannot move CUDA tensors: stage them through host memory (used
        # only to exercise the protocol; NCCL is the GPU transport)
        self.stage = dist.get_backend() == "gloo"

    def exchange(self, sends, recvs):
        """sends: [(dst, tensor)], recvs: [(src, tensor)]; batched P2P."""
        if self.stage:
            sends = [(dst, t.cpu()) for dst, t in sends]
            host = [(src, t, torch.empty(t.shape, dtype=t.dtype)) for src, t in recvs]
            ops = [self.dist.P2POp(self.dist.isend, t, dst) for dst, t in sends]
            ops += [self.dist.P2POp(self.dist.irecv, h, src) for src, _, h in host]
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            for _, t, h in host:
                t.copy_(h)
            return
        ops = [self.dist.P2POp(self.dist.isend, t, dst) for dst, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, src) for src, t in recvs]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def all_reduce_sum(self, t):
        if self.stage and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h)
            t.copy_(h)
            return t
        self.dist.all_reduce(t)
        return t


def sharded_smooth(backends, comm, K, N, world):
    """Run one time-sharded dSMC smoothing.

    backends: {rank: backend} for the ranks hosted by this process (one for
    one-process-per-GPU; all of them for in-process virtual ranks).
    comm: TorchComm, or None when every rank is hosted here.
    Returns ({rank: (mean, cov)} for the hosted windows, log Z).

    With a transport (one backend per process) every torch op of the
    protocol — the exchange tensors and the NCCL P2P calls — is issued on the
    engine's own stream, so kernel outputs and transfers are stream-ordered
    without host synchronisation.
    """
    one = backends[sorted(backends)[0]]
    if comm is not None and len(backends) == 1 and getattr(one, "stream", None) is not None:
        ctx = torch.cuda.stream(one.stream)
    else:
        ctx = contextlib.nullcontext()
    with ctx:
        out = _sharded_smooth(backends, comm, K, N, world)
    # the window moments are produced on the engine stream(s): order the
    # caller's stream after them (no host synchronisation)
    for be in backends.values():
        st = getattr(be, "stream", None)
        if st is not None:
            torch.cuda.current_stream(st.device).wait_stream(st)
    return out


def _sharded_smooth(backends, comm, K, N, world):
    """Every value of the protocol stays on the device: block log Z in a
    float64 tensor, (l, r) in int32 tensors, the window root maps composed
    with device indexing; no host synchronisation until the returned log Z.
    Virtual ranks (several backends, each on its own stream, in one
    process) hand data between streams through a host sync (`handoff`)."""
    P = world
    Kloc = K // P
    s, L = _log2(Kloc), _log2(K)
    if Kloc < 2:
        raise ValueError("each rank needs at least two leaves")
    ranks = sorted(backends)
    dev = backends[ranks[0]].comm_device
    virtual = len(backends) > 1

    def handoff():
        # virtual ranks: engines run on their own streams and torch on the
        # current one; drain both before data crosses between them
        if virtual:
            for be in backends.values():
                be.sync()
            if torch.cuda.is_available() and getattr(dev, "type", "cpu") == "cuda":
                torch.cuda.synchronize(dev)

    for g in ranks:
        backends[g].window_run(g * Kloc, Kloc)
    # log Z of every block of the current level (all ranks know all of them)
    lnc = torch.zeros(P, dtype=torch.float64, device=dev)
    cross = torch.zeros((max(P - 1, 1), 2, N), dtype=torch.int32, device=dev)
    handoff()
    for g in ranks:
        backends[g].root_lnc(lnc[g:g + 1])
    handoff()
    if comm is not None:
        comm.all_reduce_sum(lnc)
    cidx = {}
    for lev in range(s + 1, L + 1):
        span, half = 1 << lev, 1 << (lev - 1)
        nblocks = K // span
        new_lnc = torch.zeros(nblocks, dtype=torch.float64, device=dev)
        handoff()
        geo = []
        for k in range(nblocks):
            a, c, bb = k * span, k * span + half, (k + 1) * span - 1
            cidx[(lev, k)] = len(cidx)
            geo.append(dict(k=k, c=c, gA=a // Kloc, gL=(c - 1) // Kloc, gR=c // Kloc,
                            gB=bb // Kloc))
        # phase 1: right block's first-leaf slab gR -> gL
        sends, recvs, slabs = [], [], {}
        for gm in geo:
            gL, gR = gm["gL"], gm["gR"]
            if gR in backends:
                xr, colr = backends[gR].boundary(0)
                if gL in backends:
                    slabs[gm["k"]] = (xr, colr)
                else:
                    sends += [(gL, xr), (gL, colr)]
            elif gL in backends:
                xr, colr = backends[gL].empty_states(), backends[gL].empty_col()
                recvs += [(gR, xr), (gR, colr)]
                slabs[gm["k"]] = (xr, colr)
        handoff()
        if comm is not None:
            comm.exchange(sends, recvs)
        # phase 2: the cross combine on gL; l -> gA, r -> gB
        sends, recvs, remaps = [], [], []
        for gm in geo:
            k, gL = gm["k"], gm["gL"]
            if gL in backends:
                B = backends[gL]
                xl, _ = B.boundary(1)
                xr, colr = slabs[k]
                l, r = B.cross(gm["c"], lev, k, xl, xr, colr, lnc[2 * k:2 * k + 1],
                               lnc[2 * k + 1:2 * k + 2], new_lnc[k:k + 1])
                handoff()
                cross[cidx[(lev, k)], 0] = l
                cross[cidx[(lev, k)], 1] = r
                for side, dst, t in ((0, gm["gA"], l), (1, gm["gB"], r)):
                    if dst in backends:
                        remaps.append((dst, side, t))
                    else:
                        sends.append((dst, t))
            else:
                for side, dst in ((0, gm["gA"]), (1, gm["gB"])):
                    if dst in backends:
                        t = backends[dst].empty_idx()
                        recvs.append((gL, t))
                        remaps.append((dst, side, t))
        handoff()
        if comm is not None:
            comm.exchange(sends, recvs)
        for dst, side, t in remaps:
            backends[dst].remap(side, t)
        handoff()
        if comm is not None:
            comm.all_reduce_sum(new_lnc)
        lnc = new_lnc
    if comm is not None and P > 1:
        comm.all_reduce_sum(cross)
    roots = {}
    for g in ranks:
        # the window root's map through the cross levels, on the device
        t0 = g * Kloc
        M = torch.arange(N, dtype=torch.int64, device=dev)
        for lev in range(L, s, -1):
            l, r = cross[cidx[(lev, t0 >> lev)]].long()
            M = l[M] if (t0 % (1 << lev)) < (1 << (lev - 1)) else r[M]
        roots[g] = M.to(torch.int32).contiguous()
    handoff()
    out = {g: backends[g].finish(roots[g]) for g in ranks}
    handoff()
    return out, float(lnc[0])
