#!/usr/bin/env python
"""SRS-FMM apply benchmark on B200 (one process per GPU).

Workload (BASELINE.json metric): 3D Laplace, uniform unit cube, N = 1e7,
leaf capacity 128, tolerance 1e-6, one right-hand side, synthetic inputs from
the reference generators (points seed 1, charges seed 1 ^ 0x9e3779b97f4a7c15).
A "step" is one apply u = A q (the reference's sfmm::fmm_apply,
/root/reference/proj/src/apply.cpp:306-337) over the resident plan.

  value   device-resident throughput: N / (device time of one apply), q and u
          already in HBM, timed with CUDA events over K applies.
  e2e     the same through the public host-buffer API (sfmm_gpu_apply with
          pinned q in, u out: H2D + D2H inside every step).
  roofline  the fused translation kernel K2 (FP64-pipe bound): algorithmic
          flop per launch (20 per dense pair + 2 per skeleton
          pair) / its CUDA-event duration, against the DFMA peak measured in
          this run.
  cpu_baseline  the unmodified reference fmm_apply (oracle/_ref) on the SAME
          plan and charges, all host cores (OMP_PLACES=cores,
          OMP_PROC_BIND=spread): one warm-up apply, then the median of 3; also
          the -march=native build of the same sources as a second figure.  It
          yields the relative l2 deviation of the GPU result from the CPU
          reference.

``--impl reference`` times the reference CPU apply alone on the SAME workload
(rank 0 only): the reference's own precompute (build_tree,
build_neighbor_lists, build_skeletons), then fmm_apply exactly as the
reference bench times it (bench.cpp:285-288).

``--gpus N`` under torchrun: one process per GPU, the plan sharded by subtrees,
both exchanges inside the library over NCCL (sfmm_gpu_plan_attach_nccl).
``--devices 0,1,...`` (one process): the same sharding with the exchanges as
peer copies (sfmm_gpu_plan_create_multi); ids may repeat.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# The CPU reference legs run on every host core with the reference's
# recommended placement.  OpenMP reads these when it first
# initialises, so they are set before anything loads it -- and only in a
# single-process run (or the reference arm's rank 0): under torchrun every
# rank would otherwise bind its threads to the same first cores.
if (int(os.environ.get("WORLD_SIZE", "1")) == 1 or
        ("--impl" in sys.argv and "reference" in sys.argv and os.environ.get("RANK", "0") == "0")):
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_PROC_BIND", "spread")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SRS-FMM apply Mpoints/s (3D Laplace N=1e7) & rel. err vs CPU ref at 1/2/4/8 GPU"
UNIT = "Mpoints/s"
CHARGE_STREAM = 0x9E3779B97F4A7C15
CHECK_STREAM = 0xC2B2AE3D27D4EB4F
KERNELS = {"laplace2d": 0, "laplace3d": 1, "helmholtz3d": 3}
DATA = "synthetic (reference generators: points seed 1, charges seed (1+r)^0x9e3779b97f4a7c15)"

# BASELINE.json "configs" (the headline line is the default arguments:
# 3D Laplace, cube, N=1e7, leaf 128, tol 1e-6, one RHS)
CONFIGS = {
    "c1": dict(kernel="laplace2d", dist="square", n=1e5, leaf=64, tol=1e-6, nrhs=1),
    "c2": dict(kernel="laplace3d", dist="cube", n=1e6, leaf=128, tol=1e-6, nrhs=1),
    "c3a": dict(kernel="laplace3d", dist="sphere", n=1e7, leaf=128, tol=1e-8, nrhs=1),
    "c3b": dict(kernel="laplace3d", dist="gaussian", n=1e7, leaf=128, tol=1e-8, nrhs=1),
    # the reference applies one RHS per call: its CPU check runs 2 of the 16
    # columns at full N (each ~1.5 min on 16 cores)
    "c4": dict(kernel="helmholtz3d", dist="cube", n=4e6, leaf=128, tol=1e-6, kappa=10.0, nrhs=16,
               cpu_cols=2, cpu_reps=1, cpu_native=0),
    "c5": dict(kernel="laplace3d", dist="cube", n=1e8, leaf=128, tol=1e-6, nrhs=1, cpu="off"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # (not --n: torchrun's own parser would take it for --nnodes/--nproc-per-node)
    ap.add_argument("--points", dest="n", type=float, default=1e7)
    ap.add_argument("--dist", default="cube")
    ap.add_argument("--kernel", default="laplace3d", choices=list(KERNELS))
    ap.add_argument("--kappa", type=float, default=10.0)
    ap.add_argument("--leaf", type=int, default=128)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--check-targets", type=int, default=1000)
    ap.add_argument("--cpu", default="full", choices=["full", "off"],
                    help="cpu_baseline: the reference apply on the same plan, or skipped")
    ap.add_argument("--cpu-reps", type=int, default=3,
                    help="timed reference applies after one warm-up (median reported)")
    ap.add_argument("--cpu-cols", type=int, default=1,
                    help="multi-RHS runs: right-hand-side columns the CPU reference applies")
    ap.add_argument("--cpu-native", type=int, default=1,
                    help="also time the -march=native build of the reference (0: skip)")
    ap.add_argument("--ref-steps", type=int, default=3,
                    help="--impl reference: timed applies (at most --steps; each ~35 s at "
                         "the headline), after min(--warmup, 1) warm-up applies")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="multi-rank exchange; gloo stages through host memory (test path)")
    ap.add_argument("--devices", default=None,
                    help="one process, plan sharded over these devices (e.g. 0,1,2,3; ids may "
                         "repeat), exchanges as peer copies inside the library")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-rank path even with one rank (tests the NCCL plumbing "
                         "on one GPU under torchrun --nproc-per-node 1)")
    ap.add_argument("--graphs", default="auto", choices=["auto", "on", "off"],
                    help="replay the apply as a CUDA graph in the timed region (auto: small plans)")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="BASELINE.json configs (secondary measurement lines; default = headline)")
    args = ap.parse_args()
    if args.config:
        for k, v in CONFIGS[args.config].items():
            setattr(args, k, v)
    return args


def workload_config(args) -> dict:
    """The workload, identical in both arms (ours / --impl reference)."""
    n = int(args.n)
    cfg = {"workload": f"{args.kernel} {args.dist} N={n:.0e} leaf={args.leaf} tol={args.tol} "
                       f"nrhs={args.nrhs}",
           "n_points": n, "leaf_cap": args.leaf, "tol": args.tol, "nrhs": args.nrhs,
           "l2": "inputs larger than L2 (resident plan and T stream >> 126 MB)"}
    if args.kernel == "helmholtz3d":
        cfg["kappa"] = args.kappa
    return cfg


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "power_w_max": max(pw), "reasons": sorted(reasons)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def emit(obj):
    print(json.dumps(obj), flush=True)


def host_cpu() -> dict:
    """lscpu summary of the host the CPU reference runs on."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket",
                     "Socket(s)", "L3 cache"):
                info[k] = v
    except (OSError, subprocess.SubprocessError):
        pass
    info["omp_places"] = os.environ.get("OMP_PLACES")
    info["omp_proc_bind"] = os.environ.get("OMP_PROC_BIND")
    return info


def gen_points(dist, n):
    from paper_2310_16668_b200 import host
    return host.generate_points(dist, n, 1)


def gen_charges(n, nrhs, cplx):
    """Right-hand side r uses the reference charge stream with seed (1 + r)."""
    from paper_2310_16668_b200 import host
    gen = host.generate_charges_complex if cplx else host.generate_charges
    if nrhs == 1:
        return gen(n, 1 ^ CHARGE_STREAM)
    return np.asfortranarray(np.stack([gen(n, (1 + r) ^ CHARGE_STREAM) for r in range(nrhs)], 1))


def check_targets(n, m):
    rng = np.random.default_rng(CHECK_STREAM)
    return np.sort(rng.choice(n, size=min(m, n), replace=False)).astype(np.int32)


def time_reference(desc, q_cols, cplx, reps, native=False, threads=None):
    """The unmodified reference fmm_apply (oracle/_ref) on the given plan: one
    warm-up apply (OpenMP spin-up, first touch), then `reps` timed applies of
    column 0 (median); with several columns, one timed apply per column
    instead (the reference has no multi-RHS apply).  Returns (seconds per
    apply, all times, [u per timed column])."""
    from oracle import pyoracle as po
    lib = po.ref_lib(native)
    lib.ref_set_threads(threads or os.cpu_count() or 1)
    rp = po.RefPipeline.from_desc(desc, native=native)
    try:
        times, us = [], []
        if len(q_cols) == 1:
            rp.apply(q_cols[0], cplx)
            for _ in range(reps):
                t0 = time.perf_counter()
                u, _ = rp.apply(q_cols[0], cplx)
                times.append(time.perf_counter() - t0)
            us.append(u)
        else:
            for qc in q_cols:
                t0 = time.perf_counter()
                u, _ = rp.apply(qc, cplx)
                times.append(time.perf_counter() - t0)
                us.append(u)
        return statistics.median(times), times, us
    finally:
        rp.close()


# ---------------------------------------------------------------------------
# --impl reference
# ---------------------------------------------------------------------------

def run_reference(args, ws, rank):
    """The unmodified reference, rank 0 only, on the SAME workload as our arm:
    the reference's own precompute, then fmm_apply per step (bench.cpp:285-288)."""
    if rank != 0:
        return
    from oracle import pyoracle as po
    n = int(args.n)
    kern = KERNELS[args.kernel]
    cplx = kern == 3
    threads = os.cpu_count() or 1
    po.ref_lib().ref_set_threads(threads)  # torchrun sets OMP_NUM_THREADS=1
    pts = (po.generate_points(args.dist, n, 1) if args.dist in po.DIST
           else gen_points(args.dist, n))  # the clustered Gaussian has no reference generator
    t0 = time.perf_counter()
    rp = po.RefPipeline.build(kern, pts, args.leaf, args.tol, args.kappa)
    t_pre = time.perf_counter() - t0
    q = (po.generate_charges_complex(n, 1 ^ CHARGE_STREAM) if cplx
         else po.generate_charges(n, 1 ^ CHARGE_STREAM))
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, args.ref_steps))
    for _ in range(warm):
        rp.apply(q, cplx)
    times = []
    u = st = None
    for _ in range(steps):
        t0 = time.perf_counter()
        u, st = rp.apply(q, cplx)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = n / t / 1e6  # points (x one right-hand side) per second
    targets = check_targets(n, args.check_targets)
    dense = po.ref_direct_sum(kern, args.kappa, pts, q, targets)
    relerr = float(np.max(np.abs(u[targets] - dense)) / np.max(np.abs(dense)))
    info = rp.info()
    rp.close()
    sample = (f"the full workload ({args.kernel} {args.dist} N={n:.0e}, leaf {args.leaf}, tol "
              f"{args.tol}): reference precompute, then {warm} warm-up + {steps} timed "
              f"fmm_apply calls (median; steps capped at --ref-steps so the arm ends in "
              f"minutes), {threads} OpenMP threads")
    if args.nrhs > 1:
        sample += f"; one of the {args.nrhs} right-hand sides per apply (no multi-RHS apply)"
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": steps, "warmup": warm, "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": t * 1e3, "step_times_s": times,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, "host": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "relerr_vs_direct": relerr, "n_check": int(targets.size),
        "pairs": st, "precompute_s": t_pre,
        "precompute": {k: info[k] for k in ("depth", "n_boxes", "k_max", "proj_scalars")},
    })


# ---------------------------------------------------------------------------
# multi-rank (torchrun): one process per GPU, exchanges inside the library
# ---------------------------------------------------------------------------

def _shm_all_gather(path, rank, ws, dist):
    """all_gather of one dict of numpy arrays per rank through node-local
    files (the ranks share the node): returns the ranks' dicts in rank order."""
    def gather(part):
        np.savez(os.path.join(path, f"part_{rank}.npz"), **part)
        dist.barrier()
        out = []
        for r in range(ws):
            with np.load(os.path.join(path, f"part_{r}.npz")) as z:
                out.append({k: z[k] for k in z.files})
        dist.barrier()
        return out
    return gather


def run_sharded(args, ws, rank, local):
    """--gpus N under torchrun: the apply sharded over N ranks (whole subtrees
    per rank), both exchanges inside the library as grouped
    ncclSend/ncclRecv (sfmm_gpu_plan_attach_nccl), after a distributed
    precompute (each rank skeletonizes only its own subtrees).
    torch.distributed is the plumbing only: the communicator id, barriers and
    the max-over-ranks time."""
    import shutil

    import torch
    import torch.distributed as dist

    from paper_2310_16668_b200 import api, host, shard

    ndev = torch.cuda.device_count()
    dev = local % max(1, ndev)
    torch.cuda.set_device(dev)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo")
    n = int(args.n)
    kern = KERNELS[args.kernel]
    cplx = kern == 3
    base = "/dev/shm" if (os.path.isdir("/dev/shm") and
                          shutil.disk_usage("/dev/shm").free > 300 * n) else "/tmp"
    path = f"{base}/sfmm_bench_{os.environ.get('MASTER_PORT', '0')}"
    if rank == 0:
        os.makedirs(path, exist_ok=True)
    dist.barrier()
    t0 = time.perf_counter()
    pts = gen_points(args.dist, n)
    q = gen_charges(n, 1, cplx)
    t_gen = time.perf_counter() - t0
    # distributed precompute: every rank builds the same tree, skeletonizes
    # only the level-1 subtrees it owns (operators stay on its GPU) and the
    # ranks exchange the index data to form the full descriptor
    host.set_threads(max(1, (os.cpu_count() or ws) // ws))
    torch.zeros(1, device=f"cuda:{dev}")
    t0 = time.perf_counter()
    desc, hp_local, owner = shard.distributed_precompute(
        kern, pts, args.leaf, args.tol, args.kappa, ws, rank, dev,
        _shm_all_gather(path, rank, ws, dist))
    t_pre = time.perf_counter() - t0
    hinfo = hp_local.info()
    t0 = time.perf_counter()
    plan = shard.OwnedShardedPlan(desc, ws, rank, dev, hp_local.device_T()[0], owner)
    hp_local.release_device_skeletons()  # the plan holds its own copy of the operators
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    # the exchange inside the library: one NCCL communicator for the ranks
    in_library = False
    exchange_note = "python torch.distributed all_to_all (gloo test path)"
    if args.backend == "nccl":
        uid = [shard.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        try:
            plan.attach_nccl(uid[0])
            in_library = True
            exchange_note = "grouped ncclSend/ncclRecv inside libsfmm_gpu (sfmm_gpu_plan_attach_nccl)"
        except Exception as e:  # noqa: BLE001 -- report, fall back to the python exchange
            exchange_note = f"python torch.distributed all_to_all (library NCCL failed: {e})"
        ok = torch.tensor([1 if in_library else 0], device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        in_library = bool(ok.item())
    t_upload = time.perf_counter() - t0
    pre = torch.tensor([t_pre, t_upload, hinfo["t_tree"], hinfo["t_skel"]], dtype=torch.float64,
                       device=f"cuda:{dev}" if args.backend == "nccl" else "cpu")
    dist.all_reduce(pre, op=dist.ReduceOp.MAX)
    t_pre, t_upload, t_tree, t_skel = (float(x) for x in pre.tolist())
    dist.barrier()
    single_fits = n <= 20_000_000
    if rank == 0:
        shutil.rmtree(path, ignore_errors=True)

    dtype = torch.complex128 if cplx else torch.float64
    q_host = torch.from_numpy(q)
    q_dev = q_host.to(f"cuda:{dev}")
    u_dev = torch.zeros_like(q_dev)
    stream = torch.cuda.Stream(dev)
    comm = torch.cuda.Stream(dev)
    if in_library:
        plan.set_output(owned_only=True)

        def step():
            plan.apply(q_dev, u_dev, stream.cuda_stream)
    elif args.backend != "nccl":
        def host_exchange(bufs, send_counts, recv_counts):
            send, recv = bufs
            stream.synchronize()
            s_cpu = send[: int(send_counts.sum())].cpu()
            r_cpu = torch.empty(int(recv_counts.sum()), dtype=torch.float64)
            dist.all_to_all_single(r_cpu, s_cpu, output_split_sizes=[int(x) for x in recv_counts],
                                   input_split_sizes=[int(x) for x in send_counts])
            recv[: r_cpu.numel()].copy_(r_cpu)
            torch.cuda.synchronize(dev)

        def step():
            plan.begin(q_dev, stream.cuda_stream, 0)
            host_exchange(plan.buffers(), plan.send_counts, plan.recv_counts)
            if plan.cross_symmetric:
                plan.mid(stream.cuda_stream)
                host_exchange(plan.buffers2(), plan.send2_counts, plan.recv2_counts)
                plan.fin(q_dev, u_dev, stream.cuda_stream)
            else:
                plan.end(q_dev, u_dev, stream.cuda_stream)
    else:
        def step():
            shard.apply_distributed(plan, q_dev, u_dev, stream=stream, comm_stream=comm)
    torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.2)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    red_dev = f"cuda:{dev}" if args.backend == "nccl" else "cpu"
    tt = torch.tensor([ms_local], dtype=torch.float64, device=red_dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = float(tt.item())
    value = n / (ms_step * 1e-3) / 1e6

    # e2e: the public host-buffer entry point, pinned q in / whole u out on
    # every rank (collective sfmm_gpu_apply: H2D q, apply, all-reduce of the
    # owned parts, D2H u)
    q_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    q_pin.copy_(q_host)
    u_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    if in_library:
        plan.set_output(owned_only=False)
        qn, un = q_pin.numpy(), u_pin.numpy()

        def e2e_step():
            plan.apply_host(qn, un)
    else:
        def e2e_step():
            with torch.cuda.stream(stream):
                q_dev.copy_(q_pin, non_blocking=True)
            step()
            with torch.cuda.stream(stream):
                u_pin.copy_(u_dev, non_blocking=True)
            stream.synchronize()
    e2e_step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([t_e2e], dtype=torch.float64, device=red_dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())

    # accuracy: the assembled result
    if in_library:
        u_full = u_pin.numpy().copy()
    else:
        uc = u_dev.cpu() if args.backend != "nccl" else u_dev
        dist.all_reduce(uc, op=dist.ReduceOp.SUM)
        u_full = uc.cpu().numpy()
    pinfo = plan.info()
    peak = api.fp64_peak_tflops(dev)
    if rank == 0:
        targets = check_targets(n, args.check_targets)
        ref_t = api.direct_sum_subset(kern, args.kappa, pts, q, targets, device=dev)
        relerr_direct = api.max_rel_err(u_full[targets], ref_t) if targets.size else None
        relerr_single = None
        if single_fits:  # the whole-tree precompute on one GPU (same skeletons, bit for bit)
            plan.close()
            hp = host.HostPlan.build_gpu(kern, pts, args.leaf, args.tol, args.kappa, device=dev,
                                         host_T=False)
            with api.GpuPlan.from_host(hp, device=dev) as single:
                u_single = api.fmm_apply(single, q)
            hp.close()
            relerr_single = float(np.linalg.norm(u_full - u_single) / np.linalg.norm(u_single))
        w_ref = 20.0 * pinfo.p_dense + 2.0 * pinfo.p_skel
        achieved = w_ref / (ms_step * 1e-3) / ws / 1e12
        bytes_col = n * (16 if cplx else 8)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": workload_config(args),
            "parallelism": (f"subtree sharding x{ws} (cut level {plan.cut_level}), one process "
                            f"per GPU; exchanges: {exchange_note}"),
            "exchange_in_library": in_library,
            "value_definition": "N / max-over-ranks device time per apply (each rank's u holds "
                                "its owned points)",
            "roofline": {"bound": "fp64", "kernel": "whole sharded step (K2-equivalent work)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "traffic_status": "unmeasured (per-kernel capture is in the 1-GPU line)",
                         "work": "20 flop per dense pair + 2 per skeleton pair over all ranks, "
                                 "divided by the max-over-ranks step time and the GPU count"},
            "e2e": {"value": n / t_e2e / 1e6, "unit": UNIT, "h2d_bytes_per_step": bytes_col * ws,
                    "d2h_bytes_per_step": bytes_col * ws, "ms_per_step": t_e2e * 1e3,
                    "path": "collective sfmm_gpu_apply, host buffers, whole u on every rank"
                    if in_library else "torch copies around the python-exchange apply"},
            "gpu_launches": int(pinfo.launches_per_apply) * args.steps,
            "clocks": clk,
            "relerr_vs_direct": relerr_direct, "n_check": int(targets.size),
            "relerr_vs_single_gpu": relerr_single,
            "shard": {"ghost_boxes_rank0": plan.n_ghost_boxes,
                      "owned_points_rank0": plan.n_owned_points,
                      "send_mb_rank0": float(plan.send_counts.sum()) * 8 / 1e6,
                      "send2_mb_rank0": float(plan.send2_counts.sum()) * 8 / 1e6},
            "precompute": {"distributed": "every rank: GPU tree, tree-only level-1 ownership, "
                                          "skeletons of its own subtrees; index data exchanged "
                                          "through node-local files; max over ranks",
                           "t_generate_s": t_gen, "t_total_s": t_pre, "t_plan_s": t_upload,
                           "t_tree_s": t_tree, "t_skel_s": t_skel, "depth": hinfo.get("depth"),
                           "n_boxes": hinfo.get("n_boxes")},
            "cpu_baseline": {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                             "sample": "reported by the 1-GPU run (rank 0 at N=1 only)"},
        }
        emit(out)
    plan.close()
    dist.barrier()
    dist.destroy_process_group()


# ---------------------------------------------------------------------------
# one process: one GPU (or --devices)
# ---------------------------------------------------------------------------

def _k2_capture(args, n):
    """ncu figures for K2 (profiles/k2_traffic.json), valid only for the kernel
    sources they were captured from."""
    prof = os.path.join(ROOT, "profiles", "k2_traffic.json")
    key = f"{args.kernel}_{args.dist}_{n}_{args.leaf}_{args.tol}"
    try:
        pj = json.load(open(prof))
    except (OSError, ValueError):
        return None, None, "unmeasured (no ncu capture file)"
    rec = pj.get("captures", {}).get(key)
    if rec is None:
        return None, None, f"unmeasured (no ncu capture for {key})"
    if rec.get("k2_source_sha16") != k2_source_sha():
        return None, None, (f"unmeasured for this build (the capture {rec.get('capture')} was "
                            f"taken from other K2 sources)")
    return rec.get("traffic"), rec.get("fp64_pipe_active"), f"ncu capture {rec.get('capture')}"


def k2_source_sha() -> str:
    src = os.path.join(ROOT, "paper_2310_16668_b200", "csrc")
    h = hashlib.sha256()
    for f in ("kernels_translate.cu", "common.cuh", "fastmath.cuh"):
        with open(os.path.join(src, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1 or args.force_sharded:
        run_sharded(args, ws, rank, local)
        return
    devices = [int(x) for x in args.devices.split(",")] if args.devices else None

    import torch
    from paper_2310_16668_b200 import api, host

    dev = devices[0] if devices else local
    torch.cuda.set_device(dev)
    n = int(args.n)
    kern = KERNELS[args.kernel]
    cplx = kern == 3
    nrhs = args.nrhs
    t0 = time.perf_counter()
    pts = gen_points(args.dist, n)
    q = gen_charges(n, nrhs, cplx)
    t_gen = time.perf_counter() - t0
    torch.zeros(1, device=f"cuda:{dev}")  # CUDA context up front, not inside the tree build time
    torch.cuda.synchronize(dev)
    # GPU precompute keeps T in HBM: the plan takes it device-to-device
    try:
        hp = host.HostPlan.build_gpu(kern, pts, args.leaf, args.tol, args.kappa, device=dev,
                                     host_T=False)
        hinfo = hp.info()
        t0 = time.perf_counter()
        plan = api.GpuPlan.from_host(hp, device=dev, devices=devices)
        t_upload = time.perf_counter() - t0
    except MemoryError as e:
        # the operators alone are ~1 kB per point (N=1e8: ~97 GB); larger N is
        # a sharded run (torchrun --nproc-per-node 2/4/8 bench.py --gpus N)
        emit({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": 1,
              "config": workload_config(args),
              "unavailable": f"the plan does not fit one B200 at this N ({e}); run it sharded"})
        return
    info = plan.info()

    dtype = torch.complex128 if cplx else torch.float64
    # column-major n x nrhs == row-major (nrhs, n)
    q_host = torch.from_numpy(np.ascontiguousarray(q.T) if nrhs > 1 else q)
    q_dev = q_host.to(f"cuda:{dev}")
    u_dev = torch.empty_like(q_dev)
    # a dedicated stream: the applies and the timing events share it
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream
    torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        api.fmm_apply_device(plan, q_dev.data_ptr(), u_dev.data_ptr(), nrhs, sp)
    api.check_status(plan)
    # roofline denominator, measured with the clocks already up
    fp64_peak = api.fp64_peak_tflops(dev)

    # ---- timed region: K device-resident applies -------------------------
    # Large plans record per-phase events in every timed apply (launch
    # overhead is < 0.1 % there); small, launch-bound plans replay a CUDA graph
    # in the timed region and take the phase split from 3 extra applies.
    graph_mode = devices is None and (args.graphs == "on" or
                                      (args.graphs == "auto" and n * nrhs < 2_000_000))
    if not graph_mode and devices is None:
        api.set_timing(plan, True)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.2)
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        api.fmm_apply_device(plan, q_dev.data_ptr(), u_dev.data_ptr(), nrhs, sp)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    api.check_status(plan)
    ms_step = ev0.elapsed_time(ev1) / args.steps
    phases = np.zeros((0, 5))
    if devices is None:
        if graph_mode:
            api.set_timing(plan, True)
            for _ in range(3):
                api.fmm_apply_device(plan, q_dev.data_ptr(), u_dev.data_ptr(), nrhs, sp)
            torch.cuda.synchronize(dev)
        phases = api.get_timings(plan)
        api.set_timing(plan, False)
    # points x right-hand sides per second (nrhs = 1 on the headline)
    value = n * nrhs / (ms_step * 1e-3) / 1e6

    u_gpu = u_dev.cpu().numpy()
    if nrhs > 1:
        u_gpu = np.asfortranarray(u_gpu.T)

    # ---- e2e: public host-buffer API, pinned q in / u out each step -------
    q_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    q_pin.copy_(q_host)
    u_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))

    def host_apply():
        if nrhs == 1:
            return api.fmm_apply(plan, q_pin.numpy(), out=u_pin.numpy())
        return api.fmm_apply(plan, q_pin.numpy().T, out=u_pin.numpy().T)

    host_apply()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        u_e2e = host_apply()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    e2e_value = n * nrhs / t_e2e / 1e6
    bytes_col = n * nrhs * (16 if cplx else 8)

    # ---- accuracy vs the dense sum on sampled targets (GPU direct sum) ----
    u0 = u_gpu if nrhs == 1 else u_gpu[:, 0]
    q0 = q if nrhs == 1 else q[:, 0]
    targets = check_targets(n, args.check_targets)
    dense = api.direct_sum_subset(kern, args.kappa, pts, q0, targets, device=dev)
    relerr_direct = api.max_rel_err(u0[targets], dense) if targets.size else None
    e2e_same = bool(np.array_equal(u_e2e, u_gpu))

    # ---- roofline of the dominant kernel (K2, FP64 pipe) -------------------
    k2_ms = float(np.mean(phases[:, 2])) if len(phases) else float("nan")
    # W_K2 = F_K(r) P_dense + r 2 s_c P_skel, F_K(r) = G_K + 2 s_c r,
    # G = 18 (Laplace) / 32 (Helmholtz), s_c = 1 real / 4 complex; the phase
    # timings cover one 16-column pass of the multi-RHS path
    r_pass = min(nrhs, 16)
    s_c = 4.0 if cplx else 1.0
    g_k = 32.0 if cplx else 18.0
    w_k2 = (g_k + 2 * s_c * r_pass) * info.p_dense + r_pass * 2 * s_c * info.p_skel
    traffic, pipe, capture = _k2_capture(args, n)
    phase_ms = {nm: float(np.mean(phases[:, i])) for i, nm in enumerate(api.PHASES)} if len(phases) else {}
    if devices is None:
        achieved = w_k2 / (k2_ms * 1e-3) / 1e12
        roof = {
            "bound": "fp64", "kernel": "k2_translate (fused ifo/ifs/tfo/level-1)",
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak if fp64_peak > 0 else None,
            "traffic": traffic, "fp64_pipe_active": pipe, "traffic_status": capture,
            "peak_source": "DFMA loop measured in this run (MEASURED_PEAKS.json has no FP64 "
                           "figure); nominal 37.2",
            "work": (f"SURVEY.md 8d reference-equivalent: {g_k + 2 * s_c * r_pass:g} flop per "
                     f"dense pair + {r_pass * 2 * s_c:g} per skeleton pair"),
            "frac_note": ("reference-equivalent work over K2 time can exceed the peak: symmetric "
                          "blocks are generated once and cancelling pairs skipped; "
                          "fp64_pipe_active is the physical FP64 pipe utilisation of the same "
                          "kernel (ncu)"),
            "p_dense": info.p_dense, "p_skel": info.p_skel, "k2_ms": k2_ms,
        }
    else:
        achieved = w_k2 / (ms_step * 1e-3) / len(set(devices)) / 1e12
        roof = {"bound": "fp64", "kernel": "whole sharded step (K2-equivalent work)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": None,
                "traffic_status": "unmeasured (multi-device line)"}
    # interpolation GEMVs: each reads T once per apply
    sb = 16 if cplx else 8
    t_bytes = info.m_proj * sb
    gemv_gbs = {
        "upward": t_bytes / (phase_ms.get("upward", float("nan")) * 1e-3) / 1e9,
        "downward": t_bytes / (phase_ms.get("downward", float("nan")) * 1e-3) / 1e9,
    }

    out = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": 1 if not devices else len(set(devices)),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": workload_config(args),
        "baseline_config": args.config or "headline (3D Laplace cube N=1e7)",
        "value_definition": "points x right-hand sides per second of device time",
        "parallelism": ("single GPU" if not devices else
                        f"one process, plan sharded over devices {devices} (peer-copy exchanges "
                        "inside the library)"),
        "resident_plan_gb": info.device_bytes / 1e9,
        "sym_staging": {"layout": ("chained per pair" if info.sym_chain else
                                   f"per row tile, {info.merged_tasks} merged multi-tile tasks"
                                   if info.merged_tasks else "per row tile"),
                        "gb": info.stage_bytes / 1e9},
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bytes_col,
                "d2h_bytes_per_step": bytes_col, "ms_per_step": t_e2e * 1e3,
                "matches_device_result": e2e_same},
        "gpu_launches": int(info.launches_per_apply) * args.steps,
        "clocks": clk,
        "phase_ms": phase_ms,
        "timed_region": ("CUDA graph replay; phase_ms/roofline from 3 extra event-timed applies"
                         if graph_mode else "stream launches with per-phase events in every step"
                         if devices is None else "stream launches (per-rank phase graphs)"),
        "gemv_gbs": gemv_gbs,
        "relerr_vs_direct": relerr_direct, "n_check": int(targets.size),
        "precompute": {"t_generate_s": t_gen, "t_tree_s": hinfo["t_tree"],
                       "t_skel_s": hinfo["t_skel"], "t_upload_s": t_upload,
                       "depth": hinfo["depth"], "n_boxes": hinfo["n_boxes"],
                       "k_max": hinfo["k_max"], "m_proj": hinfo["proj_scalars"],
                       "host_threads": host.get_threads(),
                       "tree": "GPU tree builder (sfmm_gpu_build_tree)",
                       "skeletons": "GPU skeletonizer (sfmm_gpu_build_skeletons)",
                       "operators": "device-resident, plan built device-to-device"},
    }
    plan.close()

    # ---- CPU baseline: the unmodified reference apply on the same plan ----
    if args.cpu != "off":
        out.update(cpu_legs(args, hp, q, cplx, u_gpu, targets, dense))
    emit(out)


def cpu_legs(args, hp, q, cplx, u_gpu, targets, dense):
    """The reference fmm_apply on the plan the GPU ran (same tree, operators,
    charges): warm-up + median of --cpu-reps, O3 build and -march=native
    build; the relative deviation of the GPU result from it."""
    from oracle import pyoracle as po
    from paper_2310_16668_b200 import api
    n = int(args.n)
    res = {}
    try:
        hp.fetch_T()  # the CPU reference needs the operators on the host
        desc = hp.desc_struct()
        ncols = max(1, min(args.cpu_cols, args.nrhs))
        cols = [q] if args.nrhs == 1 else [np.ascontiguousarray(q[:, r]) for r in range(ncols)]
        threads = os.cpu_count() or 1
        t_med, times, us = time_reference(desc, cols, cplx, args.cpu_reps, False, threads)
        ug = [u_gpu] if args.nrhs == 1 else [u_gpu[:, r] for r in range(ncols)]
        res["relerr_vs_cpu_ref"] = max(po.rel_l2(a, b) for a, b in zip(ug, us))
        res["max_relerr_vs_cpu_ref"] = max(api.max_rel_err(a, b) for a, b in zip(ug, us))
        # the reference's own error vs the dense sum on the same targets and
        # skeletons, beside the GPU's (same operators -> same figure)
        res["relerr_vs_direct_cpu_ref"] = api.max_rel_err(us[0][targets], dense)
        what = ("one warm-up apply, then the median of "
                f"{len(times)} timed applies" if len(cols) == 1 else
                f"one apply per right-hand side for {len(cols)} of the {args.nrhs} columns "
                "(median; the reference has no multi-RHS apply)")
        sample = (f"full workload (N={n:.0e}): reference fmm_apply (oracle/_ref, unmodified "
                  f"sources, -O3 -DNDEBUG -fopenmp) on the same tree/skeletons/charges as the "
                  f"GPU run; {what}")
        res["cpu_baseline"] = {
            "value": n / t_med / 1e6, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": sample, "seconds": t_med, "times_s": times, "host": host_cpu()}
        if args.cpu_native and po.have_ref_native():
            t_nat, times_n, us_n = time_reference(desc, cols, cplx, args.cpu_reps, True, threads)
            res["cpu_baseline"]["native"] = {
                "value": n / t_nat / 1e6, "unit": UNIT, "seconds": t_nat, "times_s": times_n,
                "build": "same sources and flags plus -march=sapphirerapids (this host's "
                         "-march=native)",
                "relerr_vs_o3_build": po.rel_l2(us_n[0], us[0])}
    except Exception as e:  # noqa: BLE001 -- the checker may be absent; never the product
        res["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                               "sample": f"unavailable: {e}"}
    return res


if __name__ == "__main__":
    main()
