"""Time-sharded (multi-GPU) protocol: a P-rank run must reproduce the 1-rank
run exactly, because every combine keeps its global stream key.

CPU: the protocol over gloo with world_size 2 (two processes) and with
in-process virtual ranks, on the CPU test backend.
GPU: virtual ranks (one engine context each) on one GPU against the plain
single-GPU dsmc_smooth of the same model and seed, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.sharded import TorchComm, sharded_smooth

K, N, SEED = 64, 24, 17


def _model():
    return models.lgssm_check(K - 1)


def _cpu_run(P, ranks=None, comm=None, rs=abi.MULTINOMIAL):
    from oracle.py import Oracle
    from tests.sharded_cpu import CpuBackend
    m, O = _model(), Oracle()
    ranks = range(P) if ranks is None else ranks
    backends = {g: CpuBackend(m, N, SEED, O, rs) for g in ranks}
    out, lz = sharded_smooth(backends, comm, K, N, P)
    mean = torch.cat([out[g][0] for g in sorted(out)])
    return mean.numpy(), lz


def _same_lz(a, b):
    return (np.isnan(a) and np.isnan(b)) or a == b


@pytest.mark.parametrize("rs", [abi.MULTINOMIAL, abi.MH_LAZY, abi.REJECTION_LAZY])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_virtual_ranks_reproduce_single_rank_cpu(P, rs):
    m1, lz1 = _cpu_run(1, rs=rs)
    mP, lzP = _cpu_run(P, rs=rs)
    assert np.array_equal(m1, mP)
    assert _same_lz(lz1, lzP)
    assert np.isnan(lzP) == (rs != abi.MULTINOMIAL)  # lazy levels: no log Z


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mean, lz = _cpu_run(world, ranks=[rank], comm=TorchComm())
        q.put((rank, mean, lz))
    finally:
        torch.distributed.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_world_size_reproduces_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    mean = np.concatenate([r[1] for r in res])
    m1, lz1 = _cpu_run(1)
    assert np.array_equal(mean, m1)
    assert all(r[2] == lz1 for r in res)


@pytest.mark.gpu
@pytest.mark.parametrize("P,KK,NN", [(2, 256, 128), (4, 256, 128), (8, 4096, 512)])
def test_virtual_ranks_on_gpu_match_single_gpu(P, KK, NN):
    from paper_2202_02264_b200.dsmc import Engine
    from paper_2202_02264_b200.sharded import GpuBackend
    m = models.cv_tracking(KK - 1)
    ref_eng = Engine(0)
    ref = ref_eng.smooth(m, NN, abi.MULTINOMIAL, seed=SEED, precision=abi.FP32)
    engines = {g: Engine(0) for g in range(P)}
    # each rank uploads and prepares only its window (+ its right cross cut)
    backends = {g: GpuBackend(e, e.upload_window(m, g * (KK // P), KK // P), NN, m.d, SEED)
                for g, e in engines.items()}
    out, lz = sharded_smooth(backends, None, KK, NN, P)
    for b in backends.values():
        b.sync()
    mean = torch.cat([out[g][0] for g in range(P)]).cpu().numpy()
    cov = torch.cat([out[g][1] for g in range(P)]).cpu().numpy()
    assert np.array_equal(mean, ref["mean"])
    assert np.array_equal(cov, ref["cov"])
    assert lz == ref["log_norm_const"]


@pytest.mark.gpu
@pytest.mark.parametrize("rs,KK", [(abi.MH_LAZY, 1 << 12), (abi.REJECTION_LAZY, 1 << 9)])
def test_virtual_ranks_lazy_c3_shape_p8(rs, KK):
    """C3's lazy stitching across 8 windows (SV, N = 4096; K = 2^12 for
    MH-lazy B = 16, the 2^9 prefix for rejection-lazy, whose acceptance
    collapses at the trajectory's near-zero observations further on — see
    DESIGN.md): the cross combines reproduce the single-GPU run bit for bit
    (lazy resamplers could not shard)."""
    from paper_2202_02264_b200.dsmc import Engine
    from paper_2202_02264_b200.sharded import GpuBackend
    NN, P = 4096, 8
    ys = np.asarray(models.sv((1 << 16) - 1).arrays["y"], np.float64)[:KK]
    m = models.sv(KK - 1, ys=ys)
    ref = Engine(0).smooth(m, NN, rs, seed=SEED, precision=abi.FP32, mh_steps=16)
    engines = {g: Engine(0) for g in range(P)}
    backends = {g: GpuBackend(e, e.upload_window(m, g * (KK // P), KK // P), NN, m.d, SEED,
                              resampler=rs, mh_steps=16) for g, e in engines.items()}
    out, lz = sharded_smooth(backends, None, KK, NN, P)
    for b in backends.values():
        b.sync()
    mean = torch.cat([out[g][0] for g in range(P)]).cpu().numpy()
    cov = torch.cat([out[g][1] for g in range(P)]).cpu().numpy()
    assert np.array_equal(mean, ref["mean"])
    assert np.array_equal(cov, ref["cov"])
    assert np.isnan(lz) and ref["log_norm_const"] is None


def _gpu_gloo_worker(rank, world, port, q, KK, NN):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_02264_b200.dsmc import Engine
        from paper_2202_02264_b200.sharded import GpuBackend
        m = models.cv_tracking(KK - 1)
        e = Engine(0)
        be = GpuBackend(e, e.upload_window(m, rank * (KK // world), KK // world), NN, m.d, SEED)
        out, lz = sharded_smooth({rank: be}, TorchComm(), KK, NN, world)
        be.sync()
        q.put((rank, out[rank][0].cpu().numpy(), out[rank][1].cpu().numpy(), lz))
        e.close()
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.gpu
def test_process_ranks_on_gpu_match_single_gpu():
    """One process per rank through TorchComm (gloo, host-staged, both ranks
    on GPU 0) — the multi-process path bench.py takes at N > 1, with the
    protocol's torch ops on the engine stream — equals the single-GPU run."""
    from paper_2202_02264_b200.dsmc import Engine
    KK, NN, world = 1024, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_gloo_worker, args=(r, world, port, q, KK, NN))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    m = models.cv_tracking(KK - 1)
    ref = Engine(0).smooth(m, NN, abi.MULTINOMIAL, seed=SEED, precision=abi.FP32)
    assert np.array_equal(np.concatenate([r[1] for r in res]), ref["mean"])
    assert np.array_equal(np.concatenate([r[2] for r in res]), ref["cov"])
    assert all(r[3] == ref["log_norm_const"] for r in res)
