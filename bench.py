"""dSMC smoothing throughput on B200: smoothed particle-timesteps/s (T.N/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c5|c2|c1|c3]

A step is one full dSMC smoothing run (leaves -> ceil(log2 K) combine levels
-> ancestor composition -> per-time mean/cov) over the configuration's
synthetic trajectory (BASELINE.json configs; default C5: 2-D constant-velocity
LGSSM, d = 4, K = T+1 = 2^20, N = 1024, multinomial stitching, FP32 — the
north-star workload, quoted at 1/2/4/8 GPUs).

  N = 1    the whole trajectory on one GPU (dsmc_smooth_resident).
  N > 1    time-sharded (paper_2202_02264_b200/sharded.py): rank g
           owns K/N contiguous leaves and its local levels; the top log2(N)
           levels exchange boundary slabs + indices over NCCL P2P. Total work
           is fixed (scaling "strong"); results equal the 1-GPU run bit for bit.

  value  = K.N / device time per step (CUDA events on the engine stream,
           barrier + synchronize around the timed region, max over ranks),
           model resident in HBM.
  e2e    = the same metric through the public API with host (pinned) model
           arrays: H2D upload + per-time prep + run + D2H of the moments inside
           the timed region (N = 1: dsmc_smooth; N > 1: dsmc_model_upload +
           the sharded stages + D2H of the rank's window), max over ranks.
  roofline = the pair kernel (c32_pair) against the MUFU.EX2 roofline: 1 exp2
           per pair evaluation; algorithmic work = N^2 pair evaluations per
           combine x the combines of each launch, divided by the
           summed CUDA-event time of the pair launches of one step.
  cpu_baseline / --impl reference = the reference's own run_smoother compiled
           from /root/reference (oracle/_ref/libdsmc_ref.so) on all host
           threads, on a bounded sample (fewer leaves) of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(desc="C1: d=1 LGSSM (experiment.hpp lgssm-check), K=T+1=2^10, N=100, multinomial",
               model="lgssm", K=1 << 10, N=100, resampler=0),
    "c2": dict(desc="C2: 2-D constant-velocity LGSSM d=4, K=T+1=2^14, N=1024, multinomial, "
                    "RTS-marginal proposals", model="cv", K=1 << 14, N=1024, resampler=0),
    "c3": dict(desc="C3: stochastic volatility, K=T+1=2^16, N=4096, MH-lazy (B=16)",
               model="sv", K=1 << 16, N=4096, resampler=2),
    # rejection-lazy needs the exact bound of SV's stitch weight, whose
    # acceptance collapses at near-zero observations (|y_758| = 9e-5 in the
    # C3 trajectory: ~350 trials per slot over the 2^10 prefix, beyond the
    # reference's 2^24 trial cap for some seeds on longer prefixes, CPU and
    # GPU alike), so its line runs the trajectory's 2^9 prefix
    "c3r": dict(desc="C3 prefix: stochastic volatility, first K=T+1=2^9 times of the C3 "
                     "trajectory, N=4096, rejection-lazy (exact)",
                model="sv", K=1 << 9, N=4096, resampler=3, ys_len=1 << 16),
    # wide-state extension (not a BASELINE config): the N x N cross term as a
    # d-term contraction (csrc/wide.cuh), d independent AR(1) coordinates
    "c6": dict(desc="Wide-state LGSSM d=32 (32 AR(1) coordinates, rho 0.5), K=T+1=2^12, N=1024, "
                    "multinomial, RTS-marginal proposals", model="ar_iid", dim=32, K=1 << 12,
               N=1024, resampler=0),
    "c6d16": dict(desc="Wide-state LGSSM d=16, K=T+1=2^12, N=1024, multinomial",
                  model="ar_iid", dim=16, K=1 << 12, N=1024, resampler=0),
    "c6d8": dict(desc="Wide-state LGSSM d=8, K=T+1=2^12, N=1024, multinomial",
                 model="ar_iid", dim=8, K=1 << 12, N=1024, resampler=0),
    "c5": dict(desc="C5: 2-D constant-velocity LGSSM d=4, K=T+1=2^20, N=1024, multinomial, "
                    "RTS-marginal proposals", model="cv", K=1 << 20, N=1024, resampler=0),
    "c4": dict(desc="C4: SV particle Gibbs (batched c-dSMC sweep + device parameter kernel), "
                    "64 chains, K=T+1=2^12, N=512, multinomial", model="sv_pgibbs", K=1 << 12,
               N=512, resampler=0, chains=64),
}
DEFAULT_CONFIG = "c5"
# CPU sample size shared by the --impl reference arm and the cpu_baseline leg
# (runs too long for the host are timed at K' = 2^16 leaves and
# extrapolated linearly in T; dense cost is exactly T*N^2 pair evaluations)
REF_KPRIME = 1 << 16
RESAMPLERS = ["multinomial", "systematic", "mh-lazy", "rejection-lazy"]
METRIC = "smoothed particle-timesteps/sec (T·N/s)"
UNIT = "particle-timesteps/s"


def build_model(cfg, pinned=False, smoother=None):
    """smoother: the RTS used for the proposals (default: the engine's host
    RTS; the reference arm passes the oracle's so it never maps the product)."""
    from paper_2202_02264_b200 import abi, models
    T = cfg["K"] - 1
    if cfg["model"] == "cv":
        m = models.cv_tracking(T, smoother=smoother)
    elif cfg["model"] == "lgssm":
        m = models.lgssm_check(T, smoother=smoother)
    elif cfg["model"] == "ar_iid":
        m = models.ar_iid(T, cfg["dim"])
    else:
        ys = None
        if cfg.get("ys_len"):  # a prefix of the longer trajectory
            ys = np.asarray(models.sv(cfg["ys_len"] - 1).arrays["y"], np.float64)[:cfg["K"]]
        m = models.sv(T, ys=ys)
    if pinned:
        import torch
        arrays = {}
        for k, v in m.arrays.items():
            if v is None:
                arrays[k] = None
                continue
            dt = {np.float64: torch.float64, np.uint8: torch.uint8}[v.dtype.type]
            t = torch.empty(v.shape, dtype=dt, pin_memory=True)
            a = t.numpy()
            a[...] = v
            arrays[k] = a
            arrays.setdefault("_hold", []).append(t)
        hold = arrays.pop("_hold")
        kw = dict(arrays)
        if m.kind == abi.MODEL_SV:
            kw["sv"] = m.sv
        pm = abi.Model(m.kind, m.horizon, m.d, m.dy, **kw)
        pm._hold = hold
        return pm
    return m


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def bench_config(cfg, world=1):
    """The `config` object of both arms (identical, so the driver can pair
    them), including the CPU sample both arms' CPU legs run."""
    K = cfg["K"]
    c = {"workload": cfg["desc"], "K": K, "T": K - 1, "N": cfg["N"],
         "resampler": RESAMPLERS[cfg["resampler"]],
         "l2": ("inputs larger than L2 (leaf slab %.0f MB > 126 MB)" % (K * cfg["N"] * 20 * cfg.get("chains", 1) / 1e6)
                if K * cfg["N"] * 20 * cfg.get("chains", 1) > 126e6 else
                "working set %.0f MB fits in L2 (small config; no flush between steps)"
                % (K * cfg["N"] * 20 * cfg.get("chains", 1) / 1e6)),
         "parallelism": (f"time-sharded x{world} (NCCL P2P boundary exchange)" if world > 1
                         else "single GPU")}
    if "chains" in cfg:
        c["chains"] = cfg["chains"]
        c["parallelism"] = (f"chains split x{world}" if world > 1 else "single GPU")
        c["cpu_sample"] = {"K_prime": K, "chains": cfg["chains"], "extrapolated": False}
    else:
        kp = min(K, REF_KPRIME)
        c["cpu_sample"] = {"K_prime": kp, "extrapolated": kp < K,
                           "rule": "K' = min(K, 2^16) leaves, same N, d, model family; "
                                   "T*N/s extrapolated linearly in T (dense cost = T*N^2)"}
    return c


def cpu_reference(cfg):
    """One step of the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference) on all host threads: run_smoother on
    K' = min(K, 2^16) leaves with the same N, d, model family and resampler
    (C4: run_conditional for every chain, chains over threads as
    experiment.cpp:618-642). The model (RTS proposals included) is built with
    the oracle, so this process never maps the product library.
    Returns (T.N/s, cores, sample text, wall seconds)."""
    from oracle.py import Oracle, Reference
    if not Reference.available():
        return None
    R = Reference()
    threads = host_threads()
    if cfg["model"] == "sv_pgibbs":
        return cpu_reference_pgibbs(cfg, R, threads)
    Kp = min(cfg["K"], REF_KPRIME)
    m = build_model(dict(cfg, K=Kp), smoother=Oracle().kalman_smooth)
    t0 = time.perf_counter()
    r = R.run_smoother(m, cfg["N"], cfg["resampler"], seed=1 + (1 << 32), mh_steps=16,
                       threads=threads, want_paths=False)
    wall = time.perf_counter() - t0
    val = Kp * cfg["N"] / wall
    sample = (f"reference run_smoother (oracle/_ref, compiled from /root/reference) on "
              f"K'={Kp} leaves (T'={Kp - 1}), N={cfg['N']}, {RESAMPLERS[cfg['resampler']]}, "
              f"same model family, {threads} threads, wall {wall:.2f} s (RunMetadata wall "
              f"{r['wall_time_ms']:.0f} ms); "
              + ("extrapolated linearly in T to K=%d (dense cost is exactly T*N^2 pair "
                 "evaluations)" % cfg["K"] if Kp < cfg["K"] else "full workload"))
    return val, threads, sample, wall


def _pgibbs_inputs(cfg):
    from paper_2202_02264_b200 import models
    K = cfg["K"]
    ys = np.asarray(models.sv(K - 1).arrays["y"], np.float64)
    return ys, np.array([-1.0, 0.9, 0.1]), np.full(K, -1.0)


def cpu_reference_pgibbs(cfg, R, threads):
    """C4 on the CPU: the reference's run_conditional (conditional.cpp:156-216)
    for each of the chains (SV model at the chains' current theta, K = 2^12,
    N = 512, multinomial), chains spread over the host threads."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2202_02264_b200 import models
    K, N, B = cfg["K"], cfg["N"], cfg["chains"]
    ys, theta, star = _pgibbs_inputs(cfg)
    m = models.sv(K - 1, mu=theta[0], phi=theta[1], sigma=float(np.sqrt(theta[2])), ys=ys)

    def chain(c):
        return R.conditional(m, star, N, 1000 + c, 0)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(chain, range(B)))
    wall = time.perf_counter() - t0
    val = B * K * N / wall
    sample = (f"reference run_conditional (oracle/_ref, compiled from /root/reference) for "
              f"{B} chains x K={K} x N={N} (SV, multinomial), chains over {threads} host "
              f"threads, wall {wall:.2f} s; full workload, no extrapolation (the parameter "
              f"update is O(T) per chain and not timed)")
    return val, threads, sample, wall


class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", q, "--format=csv,noheader,nounits",
                                      f"--id={self.device}"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def sfu_peak_pairs_per_s(sm_max_mhz):
    """Pair-kernel peak: 1 MUFU.EX2 per pair. Measured ex2 rate if profiled
    (profiles/sfu_peak.json), else the nominal 16/clk/SM x 148 SMs."""
    p = os.path.join(ROOT, "profiles", "sfu_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["ex2_per_s"]), "measured (profiles/sfu_peak.json)"
    mhz = sm_max_mhz or 1965.0
    return 148 * 16 * mhz * 1e6, "nominal 16 ex2/clk/SM x 148 SMs at sm_max_mhz"


def _red_device(device):
    import torch
    d = torch.distributed
    if d.is_available() and d.is_initialized() and d.get_backend() == "gloo":
        return "cpu"
    return f"cuda:{device}"


def _time_steps(stream, steps, fn, world, device):
    """Barrier + synchronize, CUDA events on `stream` around exactly `steps`
    calls of fn(step), synchronize; returns the max over ranks of ms/step."""
    import torch
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for st in range(steps):
        fn(st)
    end.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([start.elapsed_time(end) / steps], device=_red_device(device))
    if world > 1:
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
    return float(ms.item())


def _max_over_ranks(v, world, device):
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_red_device(device))
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_pgibbs(args, cfg, rank, world, device):
    """C4: one step = one particle-Gibbs sweep of this rank's chains (chains
    shard across ranks: replicas, no exchange). T.N/s counts every chain."""
    import torch
    from paper_2202_02264_b200 import abi, models
    from paper_2202_02264_b200.dsmc import Engine
    torch.cuda.set_device(device)
    eng = Engine(device)
    K, N, B = cfg["K"], cfg["N"], cfg["chains"] // world
    ys, theta0, star0 = _pgibbs_inputs(cfg)
    prior = abi.SvPrior(-1.0, 1.0, 2.0, 0.2, 0.05)
    theta = torch.empty((B, 3), dtype=torch.float64, pin_memory=True).numpy()
    stars = torch.empty((B, K), dtype=torch.float64, pin_memory=True).numpy()
    theta[:] = theta0
    stars[:] = star0
    seeds = np.arange(B, dtype=np.uint64) + 1000 * (rank + 1)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=torch.device("cuda", device))

    def step(s):
        eng.sv_pgibbs_sweep(ys, theta, stars, seeds, prior, N, s)
    for w in range(args.warmup):
        step(w)
    launches0 = eng.launches
    with ClockSampler(device) as clocks:
        ms = _time_steps(stream, args.steps, lambda s: step(args.warmup + s), world, device)
    launches = eng.launches - launches0
    value = cfg["chains"] * K * N / (ms * 1e-3)
    out = None
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f32+f64 (FP32 c-dSMC, FP64 parameter kernel)",
               "data": "synthetic SV series (numpy seed 90210)",
               "config": bench_config(cfg, world),
               "e2e": {"value": value, "unit": UNIT,
                       "h2d_bytes_per_step": int(theta.nbytes + stars.nbytes + ys.nbytes),
                       "d2h_bytes_per_step": int(theta.nbytes + stars.nbytes + B * K),
                       "api": "dsmc_sv_pgibbs_sweep (C ABI) with host arrays: value is already "
                              "end to end"},
               "gpu_launches": int(launches), "clocks": clocks.summary(),
               "chain_state": {"mean_theta": theta.mean(0).tolist()}}
    eng.close()
    return out


def run_ours(args, cfg, rank, world, device):
    if cfg["model"] == "sv_pgibbs":
        return run_pgibbs(args, cfg, rank, world, device)
    import torch
    from paper_2202_02264_b200 import abi
    from paper_2202_02264_b200.dsmc import Engine
    from paper_2202_02264_b200.sharded import GpuBackend, TorchComm, sharded_smooth

    torch.cuda.set_device(device)
    eng = Engine(device)
    model = build_model(cfg, pinned=True)
    K, N, d, rs = cfg["K"], cfg["N"], model.d, cfg["resampler"]
    prec = abi.FP64_PARITY if args.precision == "fp64" else abi.FP32
    seed_base = 1 + (1 << 32)  # experiment.cpp:42-45 salting of seed 1, replicate 0
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=torch.device("cuda", device))
    h = eng.upload(model) if world == 1 else None
    eng.sync()
    if world == 1:
        def step(s):
            eng.smooth_resident(h, N, rs, seed=seed_base + s, precision=prec)
    else:
        if K % world or (K // world) < 2:
            raise SystemExit(f"K={K} does not split over {world} ranks")
        comm = TorchComm()
        # this rank's window (and its right cross cut) only
        hw = eng.upload_window(model, rank * (K // world), K // world)
        be = GpuBackend(eng, hw, N, d, seed_base, rs, device)

        def step(s):
            be.seed = seed_base + s
            return sharded_smooth({rank: be}, comm, K, N, world)
    # ---- device-resident throughput (value)
    for w in range(args.warmup):
        step(10_000 + w)
    torch.cuda.synchronize()
    launches0 = eng.launches
    with ClockSampler(device) as clocks:
        ms_max = _time_steps(stream, args.steps, step, world, device)
    launches = eng.launches - launches0
    eng.sync()  # surfaces any device error of the timed runs
    timings = eng.timings()  # last step's per-kernel-class event times
    value = K * N / (ms_max * 1e-3)
    # ---- end to end through the public API (host pinned in, host out)
    h2d = sum(a.nbytes for a in model.arrays.values() if a is not None)
    if world > 1:  # each rank uploads its window's rows (+ one cut on each side)
        h2d = int(h2d * min(1.0, (K // world + 2) / K))
    e2e_steps = max(3, min(args.steps, 10))
    if world == 1:
        d2h = K * d * 8 + K * d * d * 8 + 8
        mean_h = torch.empty((K, d), dtype=torch.float64, pin_memory=True).numpy()
        cov_h = torch.empty((K, d, d), dtype=torch.float64, pin_memory=True).numpy()

        def e2e_step(s):
            eng.smooth(model, N, rs, seed=seed_base + 5000 + s, mean_out=mean_h, cov_out=cov_h,
                       precision=prec)
    else:
        Kloc = K // world
        d2h = Kloc * (d + d * d) * 8 + 8
        mean_w = torch.empty((Kloc, d), dtype=torch.float64, pin_memory=True)
        cov_w = torch.empty((Kloc, d, d), dtype=torch.float64, pin_memory=True)

        def e2e_step(s):
            hh = eng.upload_window(model, rank * Kloc, Kloc)
            b2 = GpuBackend(eng, hh, N, d, seed_base + 5000 + s, rs, device)
            out, lz = sharded_smooth({rank: b2}, comm, K, N, world)
            mean, cov = out[rank]
            mean_w.copy_(mean)
            cov_w.copy_(cov)
            eng.free_model(hh)
    for w in range(2):  # warm (stream-ordered pool allocations)
        e2e_step(-1 - w)
    torch.cuda.synchronize()
    walls = []
    for s in range(e2e_steps):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_step(s)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    # median step (robust to a stray host hiccup), max over ranks
    e2e_s = _max_over_ranks(float(np.median(walls)), world, device)
    e2e_mean = _max_over_ranks(float(np.mean(walls)), world, device)
    e2e_val = K * N / e2e_s
    # ---- equal-precision record: the FP64 parity path (the reference's
    # operation order, bit-exact ancestors) on the same resident workload
    fp64 = None
    if world == 1 and prec == abi.FP32 and not args.no_fp64:
        f_steps = 2
        eng.smooth_resident(h, N, rs, seed=seed_base + 7000, precision=abi.FP64_PARITY)
        eng.sync()
        f_ms = _time_steps(stream, f_steps, lambda s: eng.smooth_resident(
            h, N, rs, seed=seed_base + 7001 + s, precision=abi.FP64_PARITY), world, device)
        eng.sync()
        fp64 = {"value": K * N / (f_ms * 1e-3), "unit": UNIT, "ms_per_step": f_ms,
                "steps": f_steps, "warmup": 1, "dtype": "f64",
                "note": "same workload through the FP64 parity path (reference operation "
                        "order; ancestors bit-identical to the CPU reference on the same "
                        "leaves), CUDA events on the engine stream"}
    out = None
    if rank == 0:
        ck = clocks.summary()
        pair_ms = timings[3] if len(timings) > 3 else None
        Kloc = K // world
        pairs_local = (Kloc - 1) * N * N  # rank 0's local combines (all of them at N=1)
        peak, peak_src = sfu_peak_pairs_per_s(ck.get("sm_max_mhz"))
        ach = pairs_local / (pair_ms * 1e-3) if pair_ms else None
        pk = os.environ.get("DSMC_PAIR_KERNEL", "")
        wk = os.environ.get("DSMC_WIDE_PAIR", "")
        pair_name = (("c32_prol + c32_pair_tc2 (tcgen05, opt-in)" if pk == "tc2" else
                      "c32_pair_tc (tcgen05, opt-in)" if pk == "tc" else "c32_pair") if d <= 4 else
                     "prologw_kernel + " + {"tc1": "pairw_tc_kernel", "fma": "pairw_kernel"}.get(
                         wk, "pairw_tc2_kernel") + " (tcgen05 cross term)")
        roof = {"bound": "sfu", "kernel": pair_name, "achieved": ach, "peak": peak,
                "unit": "pair-evals/s (1 MUFU.EX2 each)", "frac": ach / peak if ach else None,
                "peak_source": peak_src, "traffic": None,
                "bound_note": "the dominant kernel is bound by the special-function unit "
                              "(MUFU.EX2, one exp per pair), neither HBM nor tensor cores; "
                              "peak = measured ex2/s (DESIGN.md 5.3 for the mix ceilings)",
                "work": f"{pairs_local:.4g} pair evaluations per step on rank 0 "
                        f"({Kloc - 1} combines x N^2)",
                "pair_kernel_ms_per_step": pair_ms,
                "sample_kernel_ms_per_step": timings[4] if len(timings) > 4 else None,
                "pair_kernel_share_of_step": pair_ms / ms_max if pair_ms else None,
                "leaf_ms": timings[0], "levels_ms": timings[1],
                "compose_gather_ms": timings[2] if world == 1 else None}
        if cfg["resampler"] in (2, 3) and world == 1:
            # lazy configurations: the dominant kernel is lazy32_kernel, bound
            # by its counter-based Philox4x64-10 draws (3 u64 per MH step,
            # resampling.cpp:258-275: ceil(3 B / 4) blocks per slot and
            # combine) against the measured Philox block rate of this B200
            # (tools/philox_peak.cu -> profiles/philox_peak.json); achieved =
            # those blocks / the summed CUDA-event time of the combine levels
            # (lazy32_kernel + its per-combine finish, ~88% + ~2% of the step)
            pp = os.path.join(ROOT, "profiles", "philox_peak.json")
            ppeak = float(json.load(open(pp))["philox4x64_blocks_per_s"]) if os.path.exists(pp) else None
            B_mh = 16
            blocks = (K - 1) * N * ((3 * B_mh + 3) // 4) if cfg["resampler"] == 2 else None
            lv = timings[1]
            ach_l = blocks / (lv * 1e-3) if (blocks and lv and lv > 0) else None
            roof = {"bound": "int", "kernel": "lazy32_kernel",
                    "achieved": ach_l, "peak": ppeak, "unit": "Philox4x64-10 blocks/s",
                    "frac": (ach_l / ppeak) if (ach_l and ppeak) else None,
                    "peak_source": "measured (tools/philox_peak.cu, profiles/philox_peak.json)",
                    "traffic": None,
                    "bound_note": "lazy pair sampling is bound by its counter-based stream "
                                  "draws (integer IMAD/LOP3 work of Philox4x64-10), not by "
                                  "HBM, MUFU or tensor cores; the probe gathers hit L1/L2",
                    "work": (f"{blocks:.4g} Philox blocks per step ({K - 1} combines x N slots "
                             f"x ceil(3*{B_mh}/4))") if blocks else
                            "rejection-lazy: trials per slot are data-dependent",
                    "leaf_ms": timings[0], "levels_ms": lv,
                    "compose_gather_ms": timings[2], "levels_share_of_step": lv / ms_max}
        # HBM-class kernels: algorithmic bytes / event time
        if world == 1 and timings[0] > 0 and timings[2] > 0:
            dpb = 16 if d <= 4 else 4 * (8 if d <= 8 else 16 if d <= 16 else 32)  # state bytes
            leaf_b = K * N * (dpb + 4)           # state + column term written
            # gather: state + level-1 pair index + level-1 map (one 4-byte entry per
            # two leaves); top-down composition over levels >= 2 (sum of blocks
            # ~K/2, N entries each): map read 4 + two pair reads 8 + two writes 8
            gath_b = K * N * (dpb + 4 + 2) + (K // 2) * N * 20
            hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
                if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6551.0
            roof["hbm_kernels"] = {
                "peak_GBps": hbm,
                "leaf32": {"bytes": leaf_b, "ms": timings[0],
                           "GBps": leaf_b / (timings[0] * 1e-3) / 1e9},
                "compose_gather": {"bytes": gath_b, "ms": timings[2],
                                   "GBps": gath_b / (timings[2] * 1e-3) / 1e9}}
        # the sampler (pass 2): its MUFU work is the row log-sum-exp over the
        # sub-block sums (N * N/64 per combine) plus the recompute of <= 64
        # weights per slot (N * 64); it is latency-bound, far below that roof
        sample_ms = timings[4] if len(timings) > 4 else None
        if sample_ms and world == 1 and cfg["resampler"] in (0, 1):
            nsub = (N + 63) // 64
            ex = (K - 1) * (N * nsub + N * 64)
            roof["sfu_kernels"] = {
                "c32_sample": {"exps": ex, "ms": sample_ms,
                               "exps_per_s": ex / (sample_ms * 1e-3),
                               "frac": ex / (sample_ms * 1e-3) / peak}}
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            # traffic = DRAM bytes (read + write) per launch of the dominant
            # kernel from one ncu --set full capture; the capture's context
            # (which launch, algorithmic units per launch) in traffic_detail
            det = json.load(open(prof)).get(args.config)
            if det:
                roof["traffic"] = det.get("bytes_per_launch")
                roof["traffic_detail"] = det
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if prec == abi.FP32 else "f64",
            "data": "synthetic (trajectory simulated with numpy seed 90210; RTS-marginal proposals)",
            "config": bench_config(cfg, world),
            "precision": ("fp32 throughput path" if prec == abi.FP32 else
                          "fp64 parity path (reference operation order)"),
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                    "timing": "host wall clock per call, median of the steps (mean-based "
                              "value %.4g)" % (K * N / e2e_mean),
                    "api": ("dsmc_smooth (C ABI), host pinned arrays" if world == 1 else
                            "dsmc_model_upload + sharded window stages (C ABI), host pinned "
                            "arrays, D2H of the rank's window moments")},
            "gpu_launches": int(launches),
            "roofline": roof,
            "clocks": ck,
        }
        if fp64:
            out["fp64_parity"] = fp64
    if h is not None:
        eng.free_model(h)
    eng.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=list(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true",
                    help="skip the FP64 parity-path record of the N=1 line")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="fp64 = the bit-exact parity path (single GPU)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's CPU run_smoother on all host threads, bounded sample
        from oracle.py import Reference
        if not Reference.available():
            print(json.dumps({"impl": "reference", "unavailable":
                              "oracle/_ref/libdsmc_ref.so not built (needs /root/reference)"}))
            return
        vals, walls = [], []
        for s in range(args.warmup + args.steps):
            v, cores, sample, wall = cpu_reference(cfg)
            if s >= args.warmup:
                vals.append(v)
                walls.append(wall)
        val = float(np.median(vals))
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median(walls)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (same generator and seeds as the GPU arm)",
            "config": bench_config(cfg, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    if world > 1:
        import torch
        # one rank per GPU over NCCL; DSMC_DIST_BACKEND=gloo (host-staged, ranks
        # may share a GPU) only exercises the protocol, it is not a bench number
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        backend = os.environ.get("DSMC_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group(backend)
        # one all-rank collective before any P2P: the protocol's first
        # batch_isend_irecv then never initialises a communicator on a subset
        torch.distributed.barrier()
    out = run_ours(args, cfg, rank, world, local)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_reference(cfg)
            if cb is not None:
                v, cores, sample, wall = cb
                out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores,
                                       "kind": "reference", "sample": sample}
        print(json.dumps(out))
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
