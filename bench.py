#!/usr/bin/env python
"""Benchmark: NaivePT max-null throughput (T-matrix entries/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one full NaivePT pass over the config's synthetic input: every
permutation x voxel statistic (K0 standardise/split, K1 tcgen05 contraction
with fused t / top-2 epilogue, K2 fp64 refinement) and, for N > 1, the NCCL
all-gather of the per-permutation maxima.  Permutations are sharded across
ranks (weak in the sense of a fixed total L split N ways -> "strong").

value: whole-job T-entries/s with inputs resident in HBM (CUDA events on the
       engine's stream, max over ranks).
e2e:   the same metric through the public API (run_naive_ex / the sharded
       entry) from host numpy buffers: H2D of X, the plan's labels generated on
       the GPU (bit-identical to numpy's SFC64 shuffles, rng_kernels.cu),
       compute, D2H of maxima + argmax, all inside the timed region.
       label_gen_s reports the device label generation alone.
--impl reference: the reference algorithm's CPU implementation (the bit-exact
       C port in oracle/, all host threads) on a bounded permutation sample of
       the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "T-matrix entries/sec (perm x voxel t-stats), NaivePT max-null"
UNIT = "T-entries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rapid", action="store_true",
                    help="skip the RapidPT config-5 max-null timing (N=1)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work for the cpu_baseline sample")
    return ap.parse_args()


def progress(msg: str) -> None:
    """Phase marks on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _init_nvml(self):
        """NVML is initialised before the timed region starts (the first
        nvmlInit of a process can take longer than the whole region, which
        left a run unsampled)."""
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            return pynvml, h, mx
        except Exception:
            return None

    def _run_nvml(self) -> bool:
        """Poll NVML every 10 ms (the timed region of a step is ~35 ms)."""
        if self._nvml is None:
            return False
        pynvml, h, mx = self._nvml
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons")
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = get_reasons(h)
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.rows.append([str(self.idx), str(sm), str(mx), f"{pw:.1f}", hex(rs)] +
                                 ["Active" if rs & b else "Not Active" for b in bits])
            except Exception:
                pass
            self._stop.wait(0.01)
        return True

    def _run(self):
        if self._run_nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._nvml = self._init_nvml()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def rapid_block(device):
    """RapidPT max-null wall time at BASELINE.json config 5 (n = 400 (120/280),
    v = 524,288, L = 1e5, eta = 0.35 %, r = l = n, 50 GROUSE passes) through the
    public run_rapid API, inputs already on the host as numpy (float32-valued X):
    training (exact training columns, GROUSE, sigma / mu) + recovery (device
    Omega draws and statistics, tensor-core LS + fp64 refinement, tcgen05
    completion with Philox residuals).  A small warm-up run first loads the
    kernels.  One timed run (~17 s)."""
    import torch

    import paper_1703_01506_b200 as rmx
    from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch, scaled

    def one(cfg0, L, passes):
        x = rmx.DataMatrix(make_data_torch(cfg0, device).to(torch.float32).cpu().numpy(),
                           cfg0.n1, cfg0.n2)
        rc = rmx.RunConfig(permutations=L, seed=cfg0.plan_seed, engine="rapid",
                           training_columns=cfg0.training_columns, rank=cfg0.rank,
                           sample_rate=cfg0.sample_rate, max_passes=passes)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        null, model, counters = rmx.run_rapid(x, rc)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, null, model, counters, x

    from paper_1703_01506_b200 import rapid_engine as re

    cfg5 = CONFIGS["c5"]
    one(scaled(cfg5, (64, 64, 32), 2048), 2048, 1)  # warm-up: kernels, cuBLAS handles
    marks = [] if os.environ.get("RMX_BENCH_RAPID_MARKS") else None
    re._PHASE_LOG = marks  # device-synchronised phase marks (diagnostics only)
    try:
        dt, null, model, counters, x = one(cfg5, cfg5.permutations, 50)
    finally:
        re._PHASE_LOG = None
    L, v = cfg5.permutations, x.voxels
    return {"config": "c5: RapidPT n=400 (120/280) v=524288 L=100000 eta=0.35% r=400 "
                      "l=400, 50 GROUSE passes",
            "max_null_s": dt, "train_s": counters["train_seconds"],
            "recover_s": counters["recover_seconds"],
            "value": L * v / dt, "unit": "T-entries/s (L x v / max-null wall time)",
            "statistic_evaluations": counters["statistic_evaluations"],
            "sigma": model.residual_std, "mu": model.max_shift,
            "api": "paper_1703_01506_b200.run_rapid (host numpy in, MaxNull out)",
            **({"marks": [(tag, t - marks[0][1]) for tag, t in marks]} if marks else {})}


def cpu_sample(cfg, x_host, orders_host, seconds: float, threads: int, min_perms: int = 0):
    """Time the oracle (C port of the reference path) on a bounded sample of
    permutations of the same workload (the plan's first P, P >= min_perms);
    returns (entries/s, sample text, threads, seconds, maxima, argmax)."""
    from oracle import oracle

    v = x_host.shape[0]
    # calibrate: one permutation per thread
    p = max(1, threads)
    t0 = time.perf_counter()
    oracle.naive_maxnull(x_host, cfg.n1, orders_host[:p].astype("int64"), cfg.two_sided,
                         threads=threads)
    dt = time.perf_counter() - t0
    per_round = max(dt, 1e-6)
    rounds = max(1, int(seconds / per_round))
    P = min(orders_host.shape[0], max(p * rounds, min_perms))
    t0 = time.perf_counter()
    mx, am, _ = oracle.naive_maxnull(x_host, cfg.n1, orders_host[:P].astype("int64"),
                                     cfg.two_sided, threads=threads)
    dt = time.perf_counter() - t0
    return (P * v / dt, f"{P} permutations x {v} voxels (first {P} of the plan)", threads, dt,
            mx, am)


def _ref_import():
    """The unmodified reference package installed in baseline/_ref (pure
    Python; `pip install --target baseline/_ref /root/reference/pkg`)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "rapidmaxnull")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import rapidmaxnull

    return rapidmaxnull


def reference_numpy_naive(cfg, x_vals, perms: int = 2):
    """The reference's own numpy engine (rapidmaxnull.run_naive from
    baseline/_ref) on the plan's first `perms` permutations of the same
    workload.  Below 32 permutations its block rule (naive.py:93) makes one
    block, i.e. one thread: the rate is per core."""
    R = _ref_import()
    if R is None:
        return {"unavailable": "baseline/_ref not installed"}
    x = R.DataMatrix(x_vals, cfg.n1, cfg.n2)
    plan = R.PermutationPlan(cfg.plan_seed, perms, cfg.subjects)
    R.run_naive(x, R.PermutationPlan(cfg.plan_seed, 1, cfg.subjects), two_sided=cfg.two_sided,
                threads=1)  # warm-up (page-in, BLAS init)
    t0 = time.perf_counter()
    null, _, _ = R.run_naive(x, plan, two_sided=cfg.two_sided, threads=1)
    dt = time.perf_counter() - t0
    return {"value": perms * cfg.voxels / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "seconds": dt, "maxima": [float(m) for m in null.maxima],
            "sample": f"rapidmaxnull.run_naive (the unmodified reference, baseline/_ref) on the "
                      f"plan's first {perms} permutations x {cfg.voxels} voxels, threads=1"}


def reference_rapid_sample(x_vals, n1: int, n2: int):
    """The reference's RapidPT at config 5 (n=400 (120/280), v=524,288,
    L=1e5, eta=0.35%, r=l=400, 50 passes) timed by phase on bounded samples
    and extrapolated: one exact training column
    (tstat_full), 5 GROUSE updates (track_update on an orthonormal basis of
    the right shape -- the update's cost does not depend on its values), and
    one 32-permutation recovery span (the reference's span worker).
    Basis-init QR (one 524,288 x 400 Householder QR) is not included."""
    R = _ref_import()
    if R is None:
        return {"unavailable": "baseline/_ref not installed"}
    import numpy as np
    from rapidmaxnull import lrmc as RL
    from rapidmaxnull import rapid as RR
    from rapidmaxnull import streams as RS

    v, n = x_vals.shape
    ell = r = n
    L, passes = 100_000, 50
    k = int(np.ceil(0.0035 * v))
    x = R.DataMatrix(x_vals, n1, n2)
    plan = R.PermutationPlan(1703015065, L, n)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    x1, x2 = x.group_blocks(plan.shuffle(1))
    col = R.tstat_full(x1, x2)
    t_col = time.perf_counter() - t0
    # an orthonormal v x r basis without the 40 s QR: the first r DCT-II
    # vectors (exactly orthonormal; dense, so random row restrictions stay
    # well conditioned like a trained basis)
    i = (np.arange(v, dtype=np.float64) + 0.5) * (np.pi / v)
    u = np.cos(np.outer(i, np.arange(r, dtype=np.float64))) * np.sqrt(2.0 / v)
    u[:, 0] = 1.0 / np.sqrt(v)
    b = R.Basis(u, copy=False)
    upd = []
    for i in range(5):
        idx = np.sort(RS.stream(1703015065, RS.TRAIN_OMEGA, i, 0).choice(v, size=k, replace=False))
        t0 = time.perf_counter()
        RL.track_update(b, R.ObservedColumn(idx, col[idx]), 0.5)
        upd.append(time.perf_counter() - t0)
    t_upd = statistics.median(upd)
    model = RR.SubspaceModel(basis=b, residual_std=0.5, max_shift=0.0, training_columns=ell,
                             sample_rate=0.0035, training_maxima=np.zeros(ell), two_sided=False,
                             seed=1703015065, passes=passes, converged=False)
    # recovery: the reference's span worker (rapid.py:138-206) on a 32-permutation
    # span, one thread; the reference runs spans on `threads` workers
    # (rapid.py:232-240) -- extrapolated with ideal scaling over them
    span = 32
    out = np.empty(L)
    t0 = time.perf_counter()
    RR._recover_block(x, model, plan, ell, ell + span, k, out, [])
    t_perm = (time.perf_counter() - t0) / span
    train_s = ell * t_col + ell * passes * t_upd
    recover_s = (L - ell) * t_perm / threads
    return {"kind": "reference", "cores": threads, "extrapolated": True,
            "train_s": train_s, "recover_s": recover_s, "max_null_s": train_s + recover_s,
            "value": L * v / (train_s + recover_s), "unit": "T-entries/s (L x v / max-null time)",
            "sample": (f"rapidmaxnull (baseline/_ref) at c5 shape: 1 training column "
                       f"{t_col:.2f}s (x{ell}), median of 5 GROUSE updates {t_upd * 1e3:.0f} ms "
                       f"(x{ell * passes}), one {span}-permutation recovery span "
                       f"{t_perm * 1e3:.0f} ms/perm on one thread (x{L - ell} / {threads} "
                       f"threads, ideal scaling); basis-init QR not included")}


def _self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N ranks on this node (never silently one GPU)."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "impl": args.impl, "n_gpus": args.gpus,
                          "unavailable": f"--gpus {args.gpus} but {have} GPU(s) visible"}))
        return 2
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    import numpy as np

    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus and not (
            world == 1 and os.environ.get("RMX_BENCH_FORCE_DIST")):
        print(json.dumps({"metric": METRIC, "impl": args.impl, "n_gpus": world,
                          "unavailable": f"WORLD_SIZE={world} but --gpus={args.gpus}"}))
        return 2
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_1703_01506_b200.datagen import CONFIGS

    cfg = CONFIGS[args.config]
    v, n, L = cfg.voxels, cfg.subjects, cfg.permutations
    config_out = {"workload": f"{cfg.name}: NaivePT n={n} ({cfg.n1}/{cfg.n2}) v={v} "
                              f"grid={'x'.join(map(str, cfg.grid))} L={L} "
                              f"{'two-sided max|t|' if cfg.two_sided else 'signed max t'}",
                  "n": n, "n1": cfg.n1, "voxels": v, "permutations": L,
                  "two_sided": cfg.two_sided, "parallelism": f"perm-shard x{args.gpus}",
                  "l2": ("inputs > L2 (X 8 B x v x n + planes)" if v * n * 8 > 2 * 126e6
                         else "L2 flushed between steps (256 MB write)")}

    if args.impl == "reference":
        if rank != 0:
            return 0
        import torch  # noqa: F401  (same environment as our arm)

        from paper_1703_01506_b200.datagen import make_data_numpy, scaled
        from paper_1703_01506_b200.labels import generate_orders

        threads = os.cpu_count() or 1
        # the same workload's data (the deterministic numpy generator; the
        # statistic's cost does not depend on the values)
        small = scaled(cfg, cfg.grid, L)
        x_host = make_data_numpy(small)
        need = min(L, max(threads * 64, 256))
        orders = generate_orders(cfg.plan_seed, 0, need, n)
        vals, samples, secs = [], [], []
        for i in range(args.warmup + args.steps):
            rate, text, thr, dt, _, _ = cpu_sample(cfg, x_host, orders, args.cpu_seconds / 3,
                                                   threads)
            if i >= args.warmup:
                vals.append(rate)
                samples.append(text)
                secs.append(dt)
        value = statistics.median(vals)
        # beside the port: the reference's own numpy engine, and its RapidPT
        # at config 5 by phase (both from baseline/_ref, measured once)
        try:
            ref_np = reference_numpy_naive(cfg, x_host, perms=2)
        except Exception as exc:
            ref_np = {"unavailable": str(exc)[:200]}
        ref_rapid = None
        if not args.no_rapid:
            try:
                ref_rapid = reference_rapid_sample(x_host, 120, 280)
            except Exception as exc:
                ref_rapid = {"unavailable": str(exc)[:200]}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                # one step = one bounded sample (its measured wall time); the
                # full workload at this rate would take full_workload_s_extrapolated
                "ms_per_step": statistics.median(secs) * 1e3,
                "ms_per_step_is": "measured wall time of one bounded sample (see cpu_baseline)",
                "full_workload_s_extrapolated": v * L / value,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded smoothed Gaussian fields)",
                "config": config_out, "impl": "reference",
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                                 "sample": samples[-1] + "; bit-exact C port of the reference "
                                 "statistic path (oracle/rmx_oracle.c), all host threads"},
                "reference_numpy": {k: v_ for k, v_ in ref_np.items() if k != "maxima"},
                "rapid": ref_rapid,
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    # RMX_BENCH_FORCE_DIST=1 (tests): the multi-rank plumbing at world size 1
    dist_on = world > 1 or os.environ.get("RMX_BENCH_FORCE_DIST") == "1"
    if dist_on:
        dist.init_process_group("nccl", device_id=device)

    from paper_1703_01506_b200 import DataMatrix, PermutationPlan
    from paper_1703_01506_b200.datagen import make_data_torch
    from paper_1703_01506_b200.labels import device_orders, generate_orders
    from paper_1703_01506_b200.shard import ShardedNaive, shard_bounds

    plan = PermutationPlan(cfg.plan_seed, L, n)
    lo, hi, per = shard_bounds(L, rank, world)
    # the shard's label rows on the GPU (bit-identical to numpy's streams);
    # timed once here for the report, and again inside every e2e step
    device_orders(cfg.plan_seed, lo, min(hi, lo + 1024), n, device)  # warm the kernel
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    device_orders(cfg.plan_seed, lo, hi, n, device)
    torch.cuda.synchronize()
    label_gen_s = time.perf_counter() - t0

    x_dev = make_data_torch(cfg, device)
    torch.cuda.synchronize()
    sh = ShardedNaive(x_dev, cfg.n1, plan, cfg.two_sided)
    stream = torch.cuda.current_stream(device)

    l2_flush = None
    if x_dev.numel() * 8 < 2 * 126e6:
        l2_flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=device)

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    progress(f"rank {rank}: inputs ready, warm-up")
    for _ in range(args.warmup):
        sh.step()
    barrier()
    progress("timed steps")

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier()
        for k in range(args.steps):
            if l2_flush is not None:
                l2_flush.zero_()
            e0, e1, e2, e3 = ev[k]
            e0.record(stream)
            if sh.job is not None:
                sh.job.prepare()
                e1.record(stream)
                sh.job.tfill()
                e2.record(stream)
                sh.job.finish()
            else:
                e1.record(stream)
                e2.record(stream)
            from paper_1703_01506_b200.shard import gather_maxima

            gather_maxima(sh.job.max_out if sh.job else torch.empty(0, dtype=torch.float64,
                                                                      device=device),
                          sh.job.argmax_out if sh.job else torch.empty(0, dtype=torch.int32,
                                                                       device=device),
                          L, per)
            e3.record(stream)
        barrier()
    step_ms = [e0.elapsed_time(e3) for (e0, _, _, e3) in ev]
    tfill_ms = [e1.elapsed_time(e2) for (_, e1, e2, _) in ev]
    prep_ms = [e0.elapsed_time(e1) for (e0, e1, _, _) in ev]
    fin_ms = [e2.elapsed_time(e3) for (_, _, e2, e3) in ev]
    tot = torch.tensor([sum(step_ms) / len(step_ms), sum(tfill_ms) / len(tfill_ms)],
                       dtype=torch.float64, device=device)
    if dist_on:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step, tfill_avg = float(tot[0]), float(tot[1])
    value = L * v / (ms_per_step / 1e3)

    # ---------------- roofline of the dominant kernel (K1, tcgen05) ----------
    pk, pk_kind = peaks()
    stats0 = sh.job.stats.as_dict() if sh.job else {}
    i8 = bool(stats0.get("i8", 0))
    local_L = hi - lo
    algo_flops = 4.0 * n * v * local_L  # n MACs for S1 + n for Q1 per T entry
    achieved = algo_flops / (tfill_avg / 1e3) / 1e12
    bf16_burst = float(pk.get("bf16_tflops", 0.0) or pk.get("bf16_tflops_sustained"))
    bf16_sust = float(pk.get("bf16_tflops_sustained", bf16_burst))
    balanced = 2 * cfg.n1 == n
    i8_meas = None
    if i8:
        # u8 x s8 -> s32 MMA over K = 2 kpad (z = 255 h + l digit planes), S only.
        # Peak: the larger of 2x the measured bf16 burst (B200 dense int8 =
        # 2x dense bf16 nominally) and the int8 GEMM measured on the box
        # (cuBLASLt kind::i8, tools/measure_int8_peak.py ->
        # profiles/r02_int8_peak.json; MEASURED_PEAKS has no int8 entry)
        kpad = -(-n // 16) * 16  # the [h | l] planes share one K extent 2 kpad (32-byte MMA K step)
        exec_flops = 2.0 * (2 * kpad) * v * local_L
        peak, peak_sust = 2.0 * bf16_burst, 2.0 * bf16_sust
        peak_kind = f"{pk_kind} bf16 dense burst x 2 (int8 dense)"
        i8_meas = None
        try:
            with open(os.path.join(ROOT, "profiles", "r02_int8_peak.json")) as f:
                pj = json.load(f)
            i8_meas = {"burst": float(pj["int8_burst_tops"]),
                       "sustained": float(pj["int8_sustained_tops"]),
                       "source": "profiles/r02_int8_peak.json (cuBLASLt int8 GEMM on a B200)"}
            if i8_meas["burst"] > peak:
                peak, peak_sust = i8_meas["burst"], i8_meas["sustained"]
                peak_kind = "measured int8 dense burst (cuBLASLt)"
        except (OSError, KeyError, ValueError):
            pass
        note = ("n1 == n2: t depends on S = G.Z only; K1 runs it as an exact int8 GEMM "
                "(2 digit planes: 2 kpad int8 MACs per entry = 4 kpad ops ~ the algorithmic 4n)")
    else:
        kpad = -(-n // 16) * 16
        exec_flops = (4.0 if balanced else 8.0) * kpad * v * local_L
        peak, peak_sust = bf16_burst, bf16_sust
        peak_kind = f"{pk_kind} bf16 dense burst"
        note = ("n1 == n2: S = G.Z only, fp16 hi+lo split: 4 kpad flop per entry"
                if balanced else "S and Q, fp16 hi+lo split: 8 kpad flop per entry")
    exec_rate = exec_flops / (tfill_avg / 1e3) / 1e12
    # dram bytes of the same launch from the committed ncu capture (same
    # config, same tensor path); None when there is no capture for it
    traffic, traffic_src = None, None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                         f"r02_k1_traffic_{cfg.name}.json")
    if world == 1 and os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get("int8" if i8 else "fp16x2")
            if tj:
                traffic = float(tj["dram_bytes_read"] + tj["dram_bytes_write"])
                traffic_src = os.path.relpath(tpath, os.path.dirname(os.path.abspath(__file__)))
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per launch",
                "traffic_source": traffic_src,
                "kernel": "k_tfill_tc (K1)", "algorithmic_flops_per_launch": algo_flops,
                "algorithmic_unit": "4n flop per T entry (SURVEY 8d: n MACs for S + n for Q)",
                "kernel_ms": tfill_avg, "peak_kind": peak_kind,
                "frac_of_sustained": achieved / peak_sust,
                "executed_tensor_tflops": exec_rate, "executed_frac": exec_rate / peak,
                "tensor_path": "int8" if i8 else "fp16x2", "note": note}
    if i8 and i8_meas:
        roofline["int8_measured"] = dict(i8_meas, frac_of_burst=achieved / i8_meas["burst"],
                                         frac_of_sustained=achieved / i8_meas["sustained"])

    # ---------------- e2e through the public API from host buffers -----------
    e2e = None
    if not args.no_e2e:
        progress("e2e")
        from paper_1703_01506_b200.naive_engine import run_naive_ex

        # the configs' X is float32 (BASELINE.json); DataMatrix keeps that
        # source beside its float64 values and the engine uploads it
        x_host = DataMatrix(x_dev.to(torch.float32).cpu().numpy(), cfg.n1, cfg.n2)
        h2d_bytes = int(x_host.float32_values.nbytes)
        times = []
        first_call_s = None
        for k in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            if not dist_on:
                res = run_naive_ex(x_host, plan, two_sided=cfg.two_sided)
                _ = res.maxima
            else:
                # each rank: its permutation shard from the host X (upload
                # overlapped with K0/K1, labels generated on its GPU), then
                # the all-gather of (max, argmax)
                from paper_1703_01506_b200.shard import run_naive_distributed

                run_naive_distributed(x_host, plan, two_sided=cfg.two_sided)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if k == 0:
                first_call_s = dt  # includes page-locking X (cudaHostRegister) once
            if k >= args.warmup:
                times.append(dt)
        t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=device)
        if dist_on:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": L * v / float(t[0]), "unit": UNIT,
               "h2d_bytes_per_step": h2d_bytes,
               "x_host": "float32 v x n, page-locked (upcast to float64 on the device, exact)",
               "labels": "generated on the GPU inside the timed region (rmx_plan_orders)",
               "d2h_bytes_per_step": int(L * 12), "s_per_step": float(t[0]),
               "first_call_s": first_call_s,
               "first_call_note": "first call on a fresh host array: includes page-locking it "
                                  "in place (cudaHostRegister, amortised by later calls)",
               "api": "paper_1703_01506_b200.run_naive_ex (N=1) / run_naive_distributed (N>1)"}

    # ---------------- CPU baseline (rank 0, N=1) ------------------------------
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        progress("cpu baseline + parity")
        x_host_np = x_dev.cpu().numpy()
        threads = os.cpu_count() or 1
        orders_host = generate_orders(cfg.plan_seed, 0, min(L, max(threads * 64, 256)), n)
        try:
            rate, text, thr, dt, mx, am = cpu_sample(cfg, x_host_np, orders_host,
                                                     args.cpu_seconds, threads, min_perms=256)
            cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "port",
                   "sample": text + f" in {dt:.1f}s; bit-exact C port of the reference "
                                    "statistic path (oracle/rmx_oracle.c)"}
        except Exception as exc:  # the baseline never blocks our number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}
            mx = None
        if mx is not None:
            # the measured run's own maxima (the last timed step, same input) vs
            # the oracle's on the same permutations: bit for bit
            P = int(mx.size)
            gm = sh.job.max_out[:P].cpu().numpy()
            ga = sh.job.argmax_out[:P].cpu().numpy().astype(np.int64)
            parity = {"perms_checked": P, "voxels": v, "bit_exact": bool(np.array_equal(gm, mx)),
                      "argmax_equal": bool(np.array_equal(ga, am)),
                      "maxima_differing": int(np.sum(gm != mx)),
                      "against": "oracle/rmx_oracle.c (pinned bit-exact to the reference) on "
                                 "the benchmarked input's first permutations"}
        progress("reference numpy engine, 2 permutations")
        try:  # and the unmodified reference's own numpy engine on the first two
            rn = reference_numpy_naive(cfg, x_host_np, perms=2)
            if "maxima" in rn:
                rm = np.asarray(rn.pop("maxima"))
                parity["reference_numpy_perms_checked"] = int(rm.size)
                parity["reference_numpy_bit_exact"] = bool(
                    np.array_equal(sh.job.max_out[:rm.size].cpu().numpy(), rm))
            cpu["reference_numpy"] = rn
        except Exception as exc:
            cpu["reference_numpy"] = {"unavailable": str(exc)[:200]}

    # ---------------- RapidPT, config 5 (N=1; training is not sharded) -------
    rapid = None
    if rank == 0 and world == 1 and not args.no_rapid:
        progress("rapid (config 5)")
        try:
            rapid = rapid_block(device)
        except Exception as exc:
            rapid = {"failed": str(exc)[:200]}

    if rank == 0:
        stats = sh.job.stats.as_dict() if sh.job else {}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": ("u8 x s8 -> s32 tensor (fixed-point z, exact) + f64 refine" if i8
                      else "f16x2-split tensor (fp32 acc) + f64 refine"),
            "data": "synthetic (seeded smoothed Gaussian fields, BASELINE.json design)",
            "config": config_out,
            "clocks": clk.summary(),
            "e2e": e2e,
            # per step: K0 prep, const-reduce, K1, K2 refine; the exhaustive
            # fallback (overflow) adds exact-rows + reduce (+ transpose > 64 perms)
            "gpu_launches": args.steps * (4 + (2 + (stats0.get("overflow_perms", 0) > 64)
                                                if stats0.get("overflow_perms", 0) else 0)),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "phases_ms": {"prepare": sum(prep_ms) / len(prep_ms), "tfill": tfill_avg,
                          "finish+gather": sum(fin_ms) / len(fin_ms)},
            "engine": stats,
            "label_gen_s": label_gen_s,
            "rapid": rapid,
        }
        print(json.dumps(line))
    if dist_on:
        dist.destroy_process_group()
    if parity is not None and not (parity["bit_exact"] and parity["argmax_equal"] and
                                   parity.get("reference_numpy_bit_exact", True)):
        print("bench: the measured run's maxima differ from the oracle's", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
