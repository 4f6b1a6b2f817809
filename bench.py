#!/usr/bin/env python3
"""bench.py -- complex dd/qd MGS QR + least-squares solve on B200.

Headline workload (BASELINE.json configs[4]): batched complex quad-double
128x128 least-squares systems (a Newton-corrector batch), 4096 systems per
GPU, inputs from the reference generator (experiment.hpp:64-79; system s of
rank r draws from split_mix64(1).split(r*4096 + s)).  A "step" is one
xqr_lsq_solve_batched_device launch over the rank's 4096 systems: MGS on
[A b], y, z and the fused back substitution, all on the device.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = systems/s over all ranks, device-
resident (inputs already in HBM; the 9.6 GB working set per GPU is larger
than the 126 MB L2, so no explicit flush is needed); `e2e` = the same metric
through the host-buffer C-ABI call (xqr_lsq_solve_batched: pinned staging,
H2D of A and b, kernel, D2H of x, z and status inside the timed region).
Also reported: the single-system latency configs (configs[1..3]), the FP64
roofline of the solver kernel, the CPU baseline (the reference compiled from
/root/reference, oracle/_ref, on this host's cores) and SM clocks sampled
during the timed region.
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

METRIC = "batched complex qd MGS QR+solve (4096 x cqd 128x128 per GPU): systems/s"
UNIT = "systems/s"
FP64_PEAK_INSTR = 1.85e13  # measured FP64 lane-instr/s, profiles/r01_fp64_probe.log
FP64_PEAK_FLOPS = 36.5e12  # measured DFMA FLOP/s (fma = 2), same probe

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
    return {"workload": f"configs[4]: batched independent cqd {args.m}x{args.n} lsq_solve "
                        "(MGS on [A b] + back substitution)",
            "systems_per_gpu": per_rank, "limbs": 4, "m": args.m, "n": args.n,
            "generator": "experiment.hpp:64-79, g=1, split_mix64(1).split(rank*batch+s)",
            "l2": "inputs (9.6 GB/GPU working set) larger than L2; no flush",
            "parallelism": f"batch-sharded x{world}, no collective"}


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


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    sample = max(threads, 16)
    rates = []
    kind = "port"
    for step in range(args.warmup + args.steps):
        r, kind, dt = cpu_reference_rate(4, args.m, args.n, sample, threads,
                                         first_stream=step * sample)
        if step >= args.warmup:
            rates.append(r)
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sample / value, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64 (complex quad-double)", "data": "synthetic",
        "config": dict(arm_config(args, world, args.batch),
                       reference_sample=f"{sample} systems per step (bounded CPU sample)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} systems per step, sequential lsq_solve per system on "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm ---------------------------------------------------------------------------
def single_system_latency(xqr, ctx, torch, limbs, m, n, reps=2):
    a, b = xqr.gen_systems(limbs, 1, m, n, 1.0, 1, -1)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    dx = torch.zeros((1, n, 2, limbs), dtype=torch.float64, device="cuda")
    dz = torch.zeros((1, limbs), dtype=torch.float64, device="cuda")
    dst = torch.zeros(2, dtype=torch.int64, device="cuda")
    call = lambda: ctx.lsq_solve_batched_device(limbs, 1, m, n, da.data_ptr(), db.data_ptr(),
                                                dx.data_ptr(), dz.data_ptr(), dst.data_ptr())
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    instr, flops = work_model(limbs, m, n)
    golden = os.path.join(ROOT, "tests", "golden",
                          f"bench_{'cdd' if limbs == 2 else 'cqd'}_{m}x{n}.npz")
    parity = None
    if os.path.exists(golden):
        g = np.load(golden)
        parity = bool(np.array_equal(dx.cpu().numpy()[0].view(np.uint64), g["x"].view(np.uint64))
                      and np.array_equal(dz.cpu().numpy()[0].view(np.uint64), g["z"].view(np.uint64)))
    return {"us_per_system": ms * 1e3, "fp64_gflops": flops / (ms * 1e-3) / 1e9,
            "fp64_pipe_frac": instr / (ms * 1e-3) / FP64_PEAK_INSTR, "bitwise_vs_reference": parity}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4096, help="systems per GPU (weak scaling)")
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
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

    # one GPU per rank; BENCH_DIST_BACKEND=gloo (dev) lets a one-GPU box run
    # the N > 1 code path with every rank on the same device
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
    from paper_1210_0800_b200.sharding import max_over_ranks, shard

    limbs, m, n = 4, args.m, args.n
    first, per_rank = shard(args.batch, rank, world, args.scaling)

    ctx = xqr.Context(local)
    # one explicit stream shared by torch (events, copies) and the C ABI
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
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
    kern_ms = []
    barrier()
    e0.record()
    for _ in range(args.steps):
        step()
        kern_ms.append(None)
    e1.record()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1)
    last_kernel_ms = ctx.last_kernel_ms  # CUDA events around the last launch, ctx stream
    ms = max_over_ranks(ms, dist, red_dev)
    total = (args.batch * world if args.scaling == "weak" else args.batch) * args.steps
    value = total / (ms / 1e3)

    codes = dst.cpu().numpy()[:, 0] & 0xFFFFFFFF
    n_fail = int((codes != 0).sum())
    parity = None
    if rank == 0 and first == 0:
        ok = True
        for s in range(4):
            g = os.path.join(ROOT, "tests", "golden", f"bench_cqd_{m}x{n}_s{s}.npz")
            if not os.path.exists(g):
                ok = None
                break
            gg = np.load(g)
            ok = ok and np.array_equal(dx[s].cpu().numpy().view(np.uint64), gg["x"].view(np.uint64))
        parity = ok

    # ---- e2e through the host-buffer public API ----------------------------------------
    # inputs sit in pinned host memory (the C ABI then DMAs them directly and
    # pipelines the copies with the solves); x, z, status come back to host
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
    e2e_value = (args.batch * world if args.scaling == "weak" else args.batch) / e2e_s
    h2d = a.nbytes + b.nbytes
    d2h = xh.nbytes + zh.nbytes + 16 * per_rank

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
        if not args.no_single:
            for (L, mm, nn) in ((2, 256, 256), (4, 256, 256), (4, 512, 256)):
                single[f"{'cdd' if L == 2 else 'cqd'}_{mm}x{nn}"] = single_system_latency(
                    xqr, ctx, torch, L, mm, nn)
            # quality-up: cqd on the GPU vs cdd on one host
            # core (the reference itself), same A and b, n = 80
            try:
                import oracle  # CPU baseline leg only

                ref = oracle.reference() or oracle.port()
                gq = single_system_latency(xqr, ctx, torch, 4, 80, 80)
                a80, b80 = xqr.gen_systems(2, 1, 80, 80, 1.0, 1, -1)
                t0 = time.perf_counter()
                ref.lsq_solve(a80[0], b80[0])
                cpu_ms = 1e3 * (time.perf_counter() - t0)
                single["quality_up_n80"] = {
                    "gpu_cqd_us": gq["us_per_system"], "cpu_cdd_us_1core": cpu_ms * 1e3,
                    "speedup": cpu_ms * 1e3 / gq["us_per_system"],
                    "paper_c2050_vs_x5690": 3.08, "digits": "cqd ~62 vs cdd ~31"}
            except Exception as exc:  # noqa: BLE001
                single["quality_up_n80"] = {"unavailable": str(exc)}
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            sample = max(threads, 16)
            try:
                rate, kind, dt = cpu_reference_rate(4, m, n, sample, threads)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                       "sample": f"{sample} cqd {m}x{n} systems (streams 0..{sample - 1}), "
                                 f"sequential lsq_solve per system on {threads} threads, "
                                 f"{dt:.1f} s wall"}
            except Exception as exc:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 (complex quad-double, 4 limbs)", "data": "synthetic",
            "config": arm_config(args, world, per_rank),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d * world),
                    "d2h_bytes_per_step": int(d2h * world),
                    "api": "xqr_lsq_solve_batched (pinned host A, b -> host x, z, status; "
                           "copies pipelined with the solves)",
                    "e2e_bad_systems": int((ch != 0).sum()),
                    "e2e_matches_device": bool(np.array_equal(xh.view(np.uint64),
                                                              dx.cpu().numpy().view(np.uint64)))},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "achieved": achieved_instr / 1e12,
                         "peak": FP64_PEAK_INSTR / 1e12, "unit": "T FP64 instr/s",
                         "frac": achieved_instr / FP64_PEAK_INSTR, "traffic": traffic,
                         "kernel": "mgs_cta_kernel<L=4,LV=3,NW=8,LSQ,MINB=2> (8 warps x 2 CTAs per SM)",
                         "fp64_tflops": flops * per_rank / kernel_s / 1e12,
                         "fp64_tflops_peak": FP64_PEAK_FLOPS / 1e12,
                         "peak_source": "measured (profiles/r01_fp64_probe.log): MEASURED_PEAKS.json "
                                        "has no FP64 entry",
                         "work_per_system_instr": instr, "kernel_ms": kernel_s * 1e3,
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
