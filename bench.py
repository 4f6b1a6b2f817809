#!/usr/bin/env python3
"""bench.py -- complex dd/qd MGS QR + least-squares solve on B200.

Headline workload (BASELINE.json configs[4]): a batch of 4096 independent
complex quad-double 128x128 least-squares systems (a Newton-corrector batch)
at 1/2/4/8 GPUs.  Default scaling is STRONG: the 4096 systems are the whole
job, split into contiguous near-equal shards, rank r solving its shard with no
collective (system s always draws split_mix64(1).split(s), experiment.hpp:64-79,
so every N solves exactly the same systems).  --scaling weak gives every
rank --batch systems.  A "step" is one xqr_lsq_solve_batched_device launch
over the rank's shard: MGS on [A b], y, z and the fused back substitution.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = systems/s over all ranks, device-
resident (inputs already in HBM; the working set is larger than the 126 MB
L2, so no explicit flush is needed), timed with CUDA events and reduced with
MAX over ranks; `e2e` = the same metric through the host-buffer C-ABI call
(xqr_lsq_solve_batched: H2D of A and b, kernel, D2H of x, z and status inside
the timed region).  Also reported at N = 1: the single-system latency configs
(configs[1..3]: median of >= 20 device-resident launches after 3 warm-ups,
the median host-buffer xqr_lsq_solve latency, the reference on one host core
and its own par_lsq_solve on every core), the dd-vs-qd quality-up pair, the
FP64 roofline of the solver kernel against the FP64 peak measured live on the
same device, the CPU baseline (the reference compiled from /root/reference,
oracle/_ref, on this host's cores, with its compiler, flags and CPU model) and
SM clocks sampled during the timed region.
"""
from __future__ import annotations

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

METRIC = "batched complex qd MGS QR+solve (4096 x cqd 128x128, configs[4]): systems/s"
UNIT = "systems/s"
# fallback FP64 peak (lane-instr/s, profiles/r01_fp64_probe.log) if the live
# probe (xqr_fp64_peak, measured on the bench's own device) is unavailable
FP64_PEAK_INSTR_FALLBACK = 1.85e13

# FP64 work model: per-op instruction weights
W_DD = dict(cmul=76, cadd=40, rdiv=110, sqrt=30, cdiv=417, fma_cmul=12)
W_QD = dict(cmul=896, cadd=180, rdiv=1777, sqrt=2146, cdiv=6141, fma_cmul=40)


def work_model(limbs: int, m: int, n: int):
    """(FP64 instructions, FLOPs with fma=2) of one lsq_solve (mgs.hpp:131-158)."""
    w = W_QD if limbs == 4 else W_DD
    n_cmul = m * n * (n + 1) + m * (2 * n + 2) + n * (n - 1) // 2
    n_cadd = (2 * m - 1) * n * (n + 1) // 2 + (m - 1) * (2 * n + 2) + n * (n - 1) // 2
    n_rdiv, n_sqrt, n_cdiv = 2 * m * n, 2 * n + 2, n
    instr = (w["cmul"] * n_cmul + w["cadd"] * n_cadd + w["rdiv"] * n_rdiv + w["sqrt"] * n_sqrt
             + w["cdiv"] * n_cdiv)
    return float(instr), float(instr + w["fma_cmul"] * n_cmul)


def host_info() -> dict:
    """CPU model / cores of this host and the reference build the CPU arms load."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    info = {"cpu_model": model, "cores": os.cpu_count()}
    try:
        import oracle  # CPU baseline leg only

        info["reference_build"] = oracle.reference_build()
    except Exception as exc:  # noqa: BLE001
        info["reference_build"] = {"unavailable": str(exc)}
    return info


# ---- clocks sampled during the timed region ----------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def arm_config(args, world, per_rank):
    """The `config` both arms report (ours and --impl reference)."""
    total = args.batch if args.scaling == "strong" else args.batch * world
    return {"workload": f"configs[4]: batched independent cqd {args.m}x{args.n} lsq_solve "
                        "(MGS on [A b] + back substitution)",
            "systems_total": total, "systems_per_gpu": per_rank, "scaling": args.scaling,
            "limbs": 4, "m": args.m, "n": args.n,
            "generator": "experiment.hpp:64-79, g=1, split_mix64(1).split(s), s = global system index",
            "l2": "working set (inputs + 2.3 MB workspace per system) larger than L2; no flush",
            "parallelism": f"batch-sharded x{world} (contiguous ranges), no collective"}


# ---- the reference arm: the reference CPU implementation on this host ---------------
def cpu_reference_rate(limbs, m, n, sample, threads, seed=1, first_stream=0):
    """Reference lsq_solve (oracle/_ref = the unmodified reference headers
    compiled in place; the C restatement if that build is absent) over
    `sample` systems on `threads` host threads.  Returns (systems/s, kind)."""
    import oracle  # CPU baseline leg only

    ref = oracle.reference()
    kind = "reference"
    if ref is None:
        ref = oracle.port()
        kind = "port"
    a = np.zeros((sample, n, m, 2, limbs))
    b = np.zeros((sample, m, 2, limbs))
    for s in range(sample):
        a[s], b[s] = ref.gen_system(limbs, m, n, 1.0, seed, first_stream + s)
    t0 = time.perf_counter()
    if kind == "reference":
        x, z, codes = ref.lsq_solve_batch(a, b, threads)
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda s: ref.lsq_solve(a[s], b[s]), range(sample)))
    dt = time.perf_counter() - t0
    return sample / dt, kind, dt


CPU_SAMPLE = 256  # systems per timed reference step (a prefix of >= 256)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    rates = []
    kind = "port"
    t_total = 0.0
    for step in range(args.warmup + args.steps):
        # warm-up steps: one system per thread (caches, page faults); timed
        # steps: the bounded sample, each on fresh systems of the workload
        sample = threads if step < args.warmup else CPU_SAMPLE
        r, kind, dt = cpu_reference_rate(4, args.m, args.n, sample, threads,
                                         first_stream=(step * CPU_SAMPLE) % max(1, args.batch))
        if step >= args.warmup:
            rates.append(r)
            t_total += dt
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * CPU_SAMPLE / value, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64 (complex quad-double)", "data": "synthetic",
        "config": dict(arm_config(args, world, args.batch),
                       reference_sample=f"{CPU_SAMPLE} systems per timed step (bounded CPU sample, "
                                        "rate extrapolated to the batch)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{CPU_SAMPLE} cqd {args.m}x{args.n} systems per step, sequential "
                                   f"lsq_solve per system on {threads} threads ({t_total:.1f} s)",
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm ---------------------------------------------------------------------------
def single_system_latency(xqr, ctx, torch, limbs, m, n, reps=20, warm=3, cpu=None):
    """One single-system config (configs[1..3]): device-resident latency (the
    device-pointer entry point; median of `reps` launches after `warm`
    warm-ups, CUDA events on the ctx stream per launch), the host-buffer
    xqr_lsq_solve latency (pinned numpy in, numpy out: H2D, solve, D2H;
    median; also with pageable inputs),
    bitwise check against the reference's golden x, z, and -- with `cpu`
    (the reference build) -- the reference's lsq_solve on one host core and
    its par_lsq_solve on every core (parallel.hpp:105-153), timed once."""
    a, b = xqr.gen_systems(limbs, 1, m, n, 1.0, 1, -1)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    dx = torch.zeros((1, n, 2, limbs), dtype=torch.float64, device="cuda")
    dz = torch.zeros((1, limbs), dtype=torch.float64, device="cuda")
    dst = torch.zeros(2, dtype=torch.int64, device="cuda")
    call = lambda: ctx.lsq_solve_batched_device(limbs, 1, m, n, da.data_ptr(), db.data_ptr(),
                                                dx.data_ptr(), dz.data_ptr(), dst.data_ptr())
    for _ in range(warm):
        call()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for e0, e1 in ev:
        e0.record()
        call()
        e1.record()
    torch.cuda.synchronize()
    times = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    ms = float(np.median(times))
    instr, flops = work_model(limbs, m, n)
    golden = os.path.join(ROOT, "tests", "golden",
                          f"bench_{'cdd' if limbs == 2 else 'cqd'}_{m}x{n}.npz")
    parity = None
    if os.path.exists(golden):
        g = np.load(golden)
        parity = bool(np.array_equal(dx.cpu().numpy()[0].view(np.uint64), g["x"].view(np.uint64))
                      and np.array_equal(dz.cpu().numpy()[0].view(np.uint64), g["z"].view(np.uint64)))
    # end to end through the host-buffer public API (xqr_lsq_solve): inputs
    # in pinned host memory (as the batched e2e), x and z back into numpy
    pa = torch.from_numpy(a[0]).pin_memory().numpy()
    pb = torch.from_numpy(b[0]).pin_memory().numpy()
    for _ in range(warm):
        xqr.lsq_solve(pa, pb)
    e2e = []
    for _ in range(reps):
        t0 = time.perf_counter()
        hx, hz = xqr.lsq_solve(pa, pb)
        e2e.append(time.perf_counter() - t0)
    # the same call with pageable numpy inputs (the driver stages them)
    e2e_pg = []
    for _ in range(max(3, reps // 4)):
        t0 = time.perf_counter()
        xqr.lsq_solve(a[0], b[0])
        e2e_pg.append(time.perf_counter() - t0)
    out = {"us_per_system": ms * 1e3, "us_min": times[0] * 1e3, "us_max": times[-1] * 1e3, "reps": reps,
           "e2e_us": float(np.median(e2e)) * 1e6,
           "e2e_us_pageable_inputs": float(np.median(e2e_pg)) * 1e6,
           "fp64_gflops": flops / (ms * 1e-3) / 1e9,
           "bitwise_vs_reference": parity,
           "e2e_matches_device": bool(np.array_equal(hx.view(np.uint64), dx.cpu().numpy()[0].view(np.uint64)))}
    out["_instr"] = instr
    if cpu is not None:
        ref, threads = cpu
        t0 = time.perf_counter()
        rx, rz, st = ref.lsq_solve(a[0], b[0])
        out["cpu_ref_1core_us"] = (time.perf_counter() - t0) * 1e6
        t0 = time.perf_counter()
        px, pz, pst = ref.par_lsq_solve(a[0], b[0], threads)
        out["cpu_ref_par_us"] = (time.perf_counter() - t0) * 1e6
        out["cpu_ref_par_workers"] = threads
        out["speedup_vs_cpu_1core"] = out["cpu_ref_1core_us"] / out["us_per_system"]
        out["speedup_vs_cpu_par"] = out["cpu_ref_par_us"] / out["us_per_system"]
        out["cpu_bitwise_equal"] = bool(np.array_equal(rx.view(np.uint64), hx.view(np.uint64))
                                        and np.array_equal(px.view(np.uint64), hx.view(np.uint64)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4096,
                    help="systems in the whole job (strong) or per GPU (weak)")
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.e2e_steps = max(1, args.e2e_steps)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch

    import paper_1210_0800_b200 as xqr

    # one GPU per rank; BENCH_DIST_BACKEND=gloo (dev / tests) lets a one-GPU
    # box run the N > 1 code path with every rank on the same device
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dist = None
    red_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1210_0800_b200.sharding import max_over_ranks, shard, sum_over_ranks

    limbs, m, n = 4, args.m, args.n
    first, per_rank = shard(args.batch, rank, world, args.scaling)
    total_systems = args.batch * world if args.scaling == "weak" else args.batch

    ctx = xqr.Context(local)
    # one explicit stream shared by torch (events, copies) and the C ABI
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    # the FP64 roofline denominator, measured on this device before the run
    try:
        peak_instr = ctx.fp64_peak(0)
        peak_flops = 2.0 * ctx.fp64_peak(1)
        peak_source = "measured live on this device (xqr_fp64_peak: independent DADD / DFMA chains, " \
                      "every SM; MEASURED_PEAKS.json has no FP64 entry)"
    except Exception as exc:  # noqa: BLE001
        peak_instr, peak_flops = FP64_PEAK_INSTR_FALLBACK, 2.0 * FP64_PEAK_INSTR_FALLBACK
        peak_source = f"fallback profiles/r01_fp64_probe.log (live probe failed: {exc})"
    a, b = xqr.gen_systems(limbs, per_rank, m, n, 1.0, 1, first)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    dx = torch.zeros((per_rank, n, 2, limbs), dtype=torch.float64, device="cuda")
    dz = torch.zeros((per_rank, limbs), dtype=torch.float64, device="cuda")
    dst = torch.zeros((per_rank, 2), dtype=torch.int64, device="cuda")

    def step():
        ctx.lsq_solve_batched_device(limbs, per_rank, m, n, da.data_ptr(), db.data_ptr(),
                                     dx.data_ptr(), dz.data_ptr(), dst.data_ptr())

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1)
    last_kernel_ms = ctx.last_kernel_ms  # CUDA events around the last launch, ctx stream
    ms = max_over_ranks(ms, dist, red_dev)
    value = total_systems * args.steps / (ms / 1e3)

    codes = dst.cpu().numpy()[:, 0] & 0xFFFFFFFF
    n_fail = int(sum_over_ranks(int((codes != 0).sum()), dist, red_dev))
    parity = None
    if rank == 0 and first == 0:
        ok = True
        for s in range(min(4, per_rank)):
            g = os.path.join(ROOT, "tests", "golden", f"bench_cqd_{m}x{n}_s{s}.npz")
            if not os.path.exists(g):
                ok = None
                break
            gg = np.load(g)
            ok = ok and np.array_equal(dx[s].cpu().numpy().view(np.uint64), gg["x"].view(np.uint64))
        parity = ok

    # ---- e2e through the host-buffer public API ----------------------------------------
    # inputs sit in pinned host memory (the C ABI then DMAs them directly and
    # pipelines the copies with the solves, one kernel wave per chunk); x, z
    # and the statuses come back to host memory inside the timed region
    a_pin = torch.from_numpy(a).pin_memory().numpy()
    b_pin = torch.from_numpy(b).pin_memory().numpy()
    xqr.lsq_solve_batched(a_pin, b_pin, device=local)  # warm the workspace
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        xh, zh, ch, _ = xqr.lsq_solve_batched(a_pin, b_pin, device=local)
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    e2e_s = max_over_ranks(e2e_s, dist, red_dev)
    e2e_value = total_systems / e2e_s
    h2d = int(sum_over_ranks(a.nbytes + b.nbytes, dist, red_dev))
    d2h = int(sum_over_ranks(xh.nbytes + zh.nbytes + 16 * per_rank, dist, red_dev))
    e2e_bad = int(sum_over_ranks(int((ch != 0).sum()), dist, red_dev))
    e2e_same = bool(np.array_equal(xh.view(np.uint64), dx.cpu().numpy().view(np.uint64)))
    e2e_same = bool(sum_over_ranks(0 if e2e_same else 1, dist, red_dev) == 0)

    instr, flops = work_model(limbs, m, n)
    kernel_s = (last_kernel_ms or ms / args.steps) / 1e3
    achieved_instr = instr * per_rank / kernel_s
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"cqd_{m}x{n}_batch{per_rank}")
        except Exception:
            traffic = None
    hbm_peak = 6542.1
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass

    single = {}
    cpu = None
    if rank == 0 and world == 1:
        threads = os.cpu_count() or 1
        ref = None
        if not args.no_cpu:
            try:
                import oracle  # CPU baseline leg only

                ref = oracle.reference() or oracle.port()
            except Exception:  # noqa: BLE001
                ref = None
        if not args.no_single:
            for (L, mm, nn) in ((2, 256, 256), (4, 256, 256), (4, 512, 256)):
                r = single_system_latency(xqr, ctx, torch, L, mm, nn,
                                          cpu=(ref, threads) if ref is not None else None)
                r["fp64_pipe_frac"] = r.pop("_instr") / (r["us_per_system"] * 1e-6) / peak_instr
                single[f"{'cdd' if L == 2 else 'cqd'}_{mm}x{nn}"] = r
            # quality-up: cqd on the GPU vs cdd on one host
            # core (the reference itself), same A and b, n = 80
            if ref is not None:
                gq = single_system_latency(xqr, ctx, torch, 4, 80, 80)
                a80, b80 = xqr.gen_systems(2, 1, 80, 80, 1.0, 1, -1)
                t0 = time.perf_counter()
                ref.lsq_solve(a80[0], b80[0])
                cpu_ms = 1e3 * (time.perf_counter() - t0)
                single["quality_up_n80"] = {
                    "gpu_cqd_us": gq["us_per_system"], "cpu_cdd_us_1core": cpu_ms * 1e3,
                    "speedup": cpu_ms * 1e3 / gq["us_per_system"],
                    "paper_c2050_vs_x5690": 3.08, "digits": "cqd ~62 vs cdd ~31"}
        if ref is not None:
            try:
                rate, kind, dt = cpu_reference_rate(4, m, n, CPU_SAMPLE, threads)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                       "sample": f"{CPU_SAMPLE} cqd {m}x{n} systems (streams 0..{CPU_SAMPLE - 1}), "
                                 f"sequential lsq_solve per system on {threads} threads, "
                                 f"{dt:.1f} s wall; rate extrapolated to the batch",
                       "host": host_info()}
            except Exception as exc:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"unavailable: {exc}"}

    if rank == 0:
        waves = -(-per_rank // (2 * torch.cuda.get_device_properties(local).multi_processor_count))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 (complex quad-double, 4 limbs)", "data": "synthetic",
            "config": dict(arm_config(args, world, per_rank), kernel_waves_per_gpu=waves),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "xqr_lsq_solve_batched (pinned host A, b -> host x, z, status; "
                           "copies pipelined with the solves)",
                    "e2e_bad_systems": e2e_bad, "e2e_matches_device": e2e_same},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "achieved": achieved_instr / 1e12,
                         "peak": peak_instr / 1e12, "unit": "T FP64 instr/s",
                         "frac": achieved_instr / peak_instr, "traffic": traffic,
                         "kernel": "mgs_cta_kernel<mgs_pair<4>, NW=12, LSQ, MINB=2> (lane-pair primitives, "
                                   "12 warps x 2 CTAs per SM, 80 registers)",
                         "fp64_tflops": flops * per_rank / kernel_s / 1e12,
                         "fp64_tflops_peak": peak_flops / 1e12,
                         "peak_source": peak_source,
                         "work_per_system_instr": instr, "systems_per_launch": per_rank,
                         "kernel_ms": kernel_s * 1e3,
                         "secondary": {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak,
                                       "achieved": (traffic / kernel_s / 1e9) if traffic else None,
                                       "frac": (traffic / kernel_s / 1e9 / hbm_peak) if traffic else None,
                                       "note": "ncu dram bytes of the same launch; HBM is not the bound"}},
            "clocks": clk,
            "status": {"failed_systems": n_fail, "bitwise_vs_reference_streams_0_3": parity},
            "single_system": single,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
