#!/usr/bin/env python
"""SRS-FMM apply benchmark on B200 (one process per GPU).

Workload (BASELINE.json metric): 3D Laplace, uniform unit cube, N = 1e7,
leaf capacity 128, tolerance 1e-6, one right-hand side, synthetic inputs from
the reference generators (points seed 1, charges seed 1 ^ 0x9e3779b97f4a7c15).
A "step" is one apply u = A q (the reference's sfmm::fmm_apply,
/root/reference/proj/src/apply.cpp:306-337) over the resident plan.

  value   device-resident throughput: N / (device time of one apply), q and u
          already in HBM, timed with CUDA events over K applies.
  e2e     the same through the public host-buffer API (pinned q in, u out,
          H2D + D2H inside every step).
  roofline  the fused translation kernel K2 (FP64-pipe bound): algorithmic
          flop per launch (20 per dense pair + 2 per skeleton
          pair) / its CUDA-event duration, against the DFMA peak measured in
          this run.
  cpu_baseline  the unmodified reference fmm_apply (oracle/_ref) on the SAME
          plan and charges, all host cores, one apply; it also yields the
          relative l2 deviation of the GPU result from the CPU reference.

``--impl reference`` times the reference CPU apply alone (rank 0 only).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SRS-FMM apply Mpoints/s (3D Laplace N=1e7) & rel. err vs CPU ref at 1/2/4/8 GPU"
UNIT = "Mpoints/s"
CHARGE_STREAM = 0x9E3779B97F4A7C15
KERNELS = {"laplace2d": 0, "laplace3d": 1, "helmholtz3d": 3}


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
    ap.add_argument("--check-targets", type=int, default=1000)
    ap.add_argument("--cpu", default="full", choices=["full", "sample", "off"],
                    help="cpu_baseline: reference apply on the full plan, on the N=1e6 "
                         "instance, or skipped")
    ap.add_argument("--ref-n", type=float, default=1e6,
                    help="instance size of one --impl reference step / the 'sample' cpu baseline")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="multi-rank exchange; gloo stages through host memory (test path)")
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--graphs", default="auto", choices=["auto", "on", "off"],
                    help="replay the apply as a CUDA graph in the timed region (auto: small plans)")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="BASELINE.json configs (secondary measurement lines; default = headline)")
    args = ap.parse_args()
    if args.config:
        for k, v in CONFIGS[args.config].items():
            setattr(args, k, v)
    return args


# BASELINE.json "configs" (the headline line is the default arguments above:
# 3D Laplace, cube, N=1e7, leaf 128, tol 1e-6, one RHS)
CONFIGS = {
    "c1": dict(kernel="laplace2d", dist="square", n=1e5, leaf=64, tol=1e-6, nrhs=1),
    "c2": dict(kernel="laplace3d", dist="cube", n=1e6, leaf=128, tol=1e-6, nrhs=1),
    "c3a": dict(kernel="laplace3d", dist="sphere", n=1e7, leaf=128, tol=1e-8, nrhs=1),
    "c3b": dict(kernel="laplace3d", dist="gaussian", n=1e7, leaf=128, tol=1e-8, nrhs=1),
    "c4": dict(kernel="helmholtz3d", dist="cube", n=4e6, leaf=128, tol=1e-6, kappa=10.0, nrhs=16,
               cpu="sample", ref_n=4e5),
    "c5": dict(kernel="laplace3d", dist="cube", n=1e8, leaf=128, tol=1e-6, nrhs=1, cpu="off"),
}


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


def run_reference(args, ws, rank):
    """--impl reference: the unmodified reference CPU apply, rank 0 only."""
    if rank != 0:
        return
    from oracle import pyoracle as po
    n = int(args.ref_n)
    kern = KERNELS[args.kernel]
    if args.dist in po.DIST:
        pts = po.generate_points(args.dist, n, 1)
    else:  # clustered Gaussian (config 3b) has no reference generator
        from paper_2310_16668_b200 import host
        pts = host.generate_points(args.dist, n, 1)
    t0 = time.perf_counter()
    rp = po.RefPipeline.build(kern, pts, args.leaf, args.tol, args.kappa)
    t_pre = time.perf_counter() - t0
    cplx = kern == 3
    q = (po.generate_charges_complex(n, 1 ^ CHARGE_STREAM) if cplx
         else po.generate_charges(n, 1 ^ CHARGE_STREAM))
    for _ in range(args.warmup):
        rp.apply(q, cplx)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rp.apply(q, cplx)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = n / t / 1e6
    threads = po.ref_lib().ref_num_threads()
    sample = (f"reference fmm_apply (oracle/_ref, unmodified sources, -O3 OpenMP) on the "
              f"N={n:.0e} instance of the same workload ({args.dist}, leaf {args.leaf}, tol "
              f"{args.tol}); one apply per step, median of {args.steps}")
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators, seed 1)",
        "config": {"workload": f"{args.kernel} {args.dist} N={n:.0e} leaf={args.leaf} "
                               f"tol={args.tol} nrhs=1", "headline_n": int(args.n)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "precompute_s": t_pre,
    })


def _share_descriptor(hp, path):
    """Rank 0 writes the flat plan descriptor to node-local shared memory,
    straight from the host plan's arrays (no intermediate copy: at N=1e8 T alone
    is ~100 GB)."""
    import ctypes as C
    from paper_2310_16668_b200._abi import DESC_ARRAYS, DESC_SCALARS, _array_len
    st = hp.desc_struct()
    sc = {k: getattr(st, k) for k in DESC_SCALARS}
    os.makedirs(path, exist_ok=True)
    views = {}
    for name, dt in [(n, d) for n, d in DESC_ARRAYS if n.endswith("_off")] + \
                    [(n, d) for n, d in DESC_ARRAYS if not n.endswith("_off")]:
        cnt = _array_len(name, sc, lambda k: views[k])
        ptr = getattr(st, name)
        views[name] = (np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                             shape=(cnt,)) if cnt and ptr else np.zeros(0, dtype=dt))
        np.save(os.path.join(path, name + ".npy"), views[name])
    with open(os.path.join(path, "scalars.json"), "w") as f:
        json.dump(sc, f)


def _load_descriptor(path):
    from paper_2310_16668_b200._abi import DESC_ARRAYS, PlanDescriptor
    arrays = {n: np.load(os.path.join(path, n + ".npy"), mmap_mode="r") for n, _ in DESC_ARRAYS}
    with open(os.path.join(path, "scalars.json")) as f:
        scalars = json.load(f)
    return PlanDescriptor(scalars, arrays)


def run_sharded(args, ws, rank, local):
    """--gpus N under torchrun: strong scaling of the N=1e7 headline apply over
    N ranks, whole level-1 subtrees per rank, ghost all-to-all over NCCL after
    the upward pass, one translation launch."""
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
    # node-local shared memory for the descriptor (~0.1 kB per point without T, ~1.3 kB
    # with it), else /tmp
    per_point = 300
    base = "/dev/shm" if (os.path.isdir("/dev/shm") and
                          shutil.disk_usage("/dev/shm").free > per_point * n) else "/tmp"
    path = f"{base}/sfmm_bench_{os.environ.get('MASTER_PORT', '0')}"
    t0 = time.perf_counter()
    pts = host.generate_points(args.dist, n, 1)
    q = (host.generate_charges_complex(n, 1 ^ CHARGE_STREAM) if cplx
         else host.generate_charges(n, 1 ^ CHARGE_STREAM))
    hp = None
    hinfo = {}
    device_T = True
    if rank == 0:
        # torchrun sets OMP_NUM_THREADS=1; the other ranks wait at the barrier
        host.set_threads(os.cpu_count() or 1)
        # GPU precompute keeps T on rank 0's device: the descriptor is shared
        # without it and every rank receives only its own operators (NCCL)
        hp = host.HostPlan.build_gpu(kern, pts, args.leaf, args.tol, args.kappa, device=dev,
                                     host_T=False)
        hinfo = hp.info()
        _share_descriptor(hp, path)
    dist.barrier()
    if rank != 0:
        host.set_threads(max(1, (os.cpu_count() or ws) // ws))
    desc = hp.desc_struct() if rank == 0 else _load_descriptor(path)
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    blob = None
    if device_T:
        sw = 2 if cplx else 1
        runs, n_entries = shard.T_runs(desc, ws, rank)
        all_runs = [None] * ws
        dist.all_gather_object(all_runs, runs)
        blob = torch.empty(max(1, n_entries * sw), dtype=torch.float64, device=f"cuda:{dev}")
        if rank == 0:
            ptr, _, _ = hp.device_T()
            for r in range(ws):
                if r == 0:
                    shard.pack_T(ptr, all_runs[0], sw, blob, dev)
                    continue
                cnt = max(1, int(all_runs[r][:, 1].sum()) * sw)
                buf = torch.empty(cnt, dtype=torch.float64, device=f"cuda:{dev}")
                shard.pack_T(ptr, all_runs[r], sw, buf, dev)
                torch.cuda.synchronize(dev)
                dist.send(buf if args.backend == "nccl" else buf.cpu(), dst=r)
                del buf
        else:
            if args.backend == "nccl":
                dist.recv(blob, src=0)
            else:
                tmp = torch.empty(blob.numel(), dtype=torch.float64)
                dist.recv(tmp, src=0)
                blob.copy_(tmp)
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()  # rank 0's pack buffers: give the plan its memory back
    plan = shard.ShardedPlan(desc, ws, rank, device=dev, T_owned=blob)
    del blob
    torch.cuda.empty_cache()
    t_upload = time.perf_counter() - t0
    dist.barrier()
    # the single-GPU parity check below needs the full operators on rank 0
    single_fits = n <= 20_000_000
    if rank == 0:
        shutil.rmtree(path, ignore_errors=True)
        if device_T and not single_fits:
            hp.release_device_skeletons()

    dtype = torch.complex128 if cplx else torch.float64
    q_host = torch.from_numpy(q)
    q_dev = q_host.to(f"cuda:{dev}")
    u_dev = torch.zeros_like(q_dev)
    stream = torch.cuda.Stream(dev)
    comm = torch.cuda.Stream(dev)
    if args.backend != "nccl":
        # test path (several ranks on one GPU): exchange through host memory
        def host_exchange(bufs, send_counts, recv_counts):
            send, recv = bufs
            stream.synchronize()
            s_cpu = send[: int(send_counts.sum())].cpu()
            r_cpu = torch.empty(int(recv_counts.sum()), dtype=torch.float64)
            dist.all_to_all_single(r_cpu, s_cpu, output_split_sizes=[int(x) for x in recv_counts],
                                   input_split_sizes=[int(x) for x in send_counts])
            recv[: r_cpu.numel()].copy_(r_cpu)
            torch.cuda.synchronize(dev)

        def exchange_apply():
            plan.begin(q_dev, stream.cuda_stream, 0)
            host_exchange(plan.buffers(), plan.send_counts, plan.recv_counts)
            if plan.cross_symmetric:
                plan.mid(stream.cuda_stream)
                host_exchange(plan.buffers2(), plan.send2_counts, plan.recv2_counts)
                plan.fin(q_dev, u_dev, stream.cuda_stream)
            else:
                plan.end(q_dev, u_dev, stream.cuda_stream)
    else:
        def exchange_apply():
            shard.apply_distributed(plan, q_dev, u_dev, stream=stream, comm_stream=comm)
    torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        exchange_apply()
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
        exchange_apply()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    tt = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{dev}" if args.backend == "nccl" else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = float(tt.item())
    value = n / (ms_step * 1e-3) / 1e6

    # e2e: pinned q -> device, apply, device u -> pinned host, every step
    q_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    q_pin.copy_(q_host)
    u_pin = torch.empty(q_host.shape, dtype=dtype).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        with torch.cuda.stream(stream):
            q_dev.copy_(q_pin, non_blocking=True)
        exchange_apply()
        with torch.cuda.stream(stream):
            u_pin.copy_(u_dev, non_blocking=True)
        stream.synchronize()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([t_e2e], dtype=torch.float64, device=tt.device)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())

    # accuracy: assemble the owned slices (all other entries are zero)
    if args.backend == "nccl":
        dist.all_reduce(u_dev, op=dist.ReduceOp.SUM)
        u_full = u_dev.cpu().numpy()
    else:
        uc = u_dev.cpu()
        dist.all_reduce(uc, op=dist.ReduceOp.SUM)
        u_full = uc.numpy()
    out = None
    pinfo = plan.info()
    peak = api.fp64_peak_tflops(dev)
    if rank == 0:
        rng = np.random.default_rng(0xC2B2AE3D27D4EB4F)
        targets = np.sort(rng.choice(n, size=min(args.check_targets, n), replace=False)).astype(np.int32)
        ref_t = api.direct_sum_subset(kern, args.kappa, pts, q, targets, device=dev)
        relerr_direct = api.max_rel_err(u_full[targets], ref_t) if targets.size else None
        # parity of the sharded result against the single-GPU plan (same operators)
        relerr_single = None
        if single_fits:
            with (api.GpuPlan.from_host(hp, device=dev) if device_T else
                  api.GpuPlan(desc, device=dev)) as single:
                u_single = api.fmm_apply(single, q)
            relerr_single = float(np.linalg.norm(u_full - u_single) / np.linalg.norm(u_single))
        # whole-job reference-equivalent K2 work over the step time, per GPU
        w_ref = 20.0 * pinfo.p_dense + 2.0 * pinfo.p_skel
        achieved = w_ref / (ms_step * 1e-3) / ws / 1e12
        bytes_col = n * (16 if cplx else 8)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generators: points seed 1, charges seed 1^0x9e3779b97f4a7c15)",
            "config": {
                "workload": f"{args.kernel} {args.dist} N={n:.0e} leaf={args.leaf} tol={args.tol} nrhs=1",
                "n_points": n, "leaf_cap": args.leaf, "tol": args.tol, "nrhs": 1,
                "parallelism": (f"subtree sharding x{ws} (cut level {plan.cut_level}), ghost and "
                                f"column-sum all-to-alls over {args.backend}"),
                "l2": "inputs larger than L2",
            },
            "roofline": {"bound": "fp64", "kernel": "whole sharded step (K2-equivalent work)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "work": "20 flop per dense pair + 2 per skeleton pair over all ranks, "
                                 "divided by the max-over-ranks step time and the GPU count; the "
                                 "per-kernel roofline is in the 1-GPU line"},
            "e2e": {"value": n / t_e2e / 1e6, "unit": UNIT, "h2d_bytes_per_step": bytes_col * ws,
                    "d2h_bytes_per_step": bytes_col * ws, "ms_per_step": t_e2e * 1e3},
            # rank 0 per apply: the single-RHS sequence plus ghost pack / unpack and the
            # column-sum pack (plan_info counts them for sharded plans)
            "gpu_launches": int(pinfo.launches_per_apply) * args.steps,
            "clocks": clk,
            "relerr_vs_direct": relerr_direct, "n_check": int(targets.size),
            "relerr_vs_single_gpu": relerr_single,
            "shard": {"ghost_boxes_rank0": plan.n_ghost_boxes,
                      "owned_points_rank0": plan.n_owned_points,
                      "send_mb_rank0": float(plan.send_counts.sum()) * 8 / 1e6,
                      "send2_mb_rank0": float(plan.send2_counts.sum()) * 8 / 1e6},
            "precompute": {"t_total_s": t_pre, "t_upload_s": t_upload, **{k: hinfo.get(k) for k in
                           ("depth", "n_boxes", "k_max", "t_tree", "t_skel")}},
            "cpu_baseline": {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                             "sample": "reported by the 1-GPU run (rank 0 at N=1 only)"},
        }
        emit(out)
    plan.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1:
        run_sharded(args, ws, rank, local)
        return
    if args.n > 6e7:
        # ~1.8 kB of resident plan per point (T, staging, slots): N=1e8 needs
        # ~180 GB, more than one B200 -- config 5 is a 2/4/8-GPU sharded run
        emit({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": 1,
              "config": {"workload": f"{args.kernel} {args.dist} N={args.n:.0e}"},
              "unavailable": "the resident plan exceeds one B200's HBM at this N; run it sharded "
                             "(torchrun --nproc-per-node 2/4/8 bench.py --gpus N --config c5)"})
        return

    import torch
    from paper_2310_16668_b200 import api, host

    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = local

    n = int(args.n)
    kern = KERNELS[args.kernel]
    cplx = kern == 3
    nrhs = args.nrhs
    t0 = time.perf_counter()
    pts = host.generate_points(args.dist, n, 1)
    # right-hand side r uses the reference charge stream with seed (1 + r)
    gen = host.generate_charges_complex if cplx else host.generate_charges
    q = gen(n, 1 ^ CHARGE_STREAM)
    if nrhs > 1:
        q = np.asfortranarray(np.stack([gen(n, (1 + r) ^ CHARGE_STREAM) for r in range(nrhs)], 1))
    t_gen = time.perf_counter() - t0
    torch.zeros(1, device=f"cuda:{dev}")  # CUDA context up front, not inside the tree build time
    torch.cuda.synchronize(dev)
    # GPU precompute keeps T in HBM: the plan takes it device-to-device
    hp = host.HostPlan.build_gpu(kern, pts, args.leaf, args.tol, args.kappa, device=dev,
                                 host_T=False)
    hinfo = hp.info()
    t0 = time.perf_counter()
    plan = api.GpuPlan.from_host(hp, device=dev)
    t_upload = time.perf_counter() - t0
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
    graph_mode = args.graphs == "on" or (args.graphs == "auto" and n * nrhs < 2_000_000)
    if not graph_mode:
        api.set_timing(plan, True)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.2)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        api.fmm_apply_device(plan, q_dev.data_ptr(), u_dev.data_ptr(), nrhs, sp)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    api.check_status(plan)
    ms_step = ev0.elapsed_time(ev1) / args.steps
    if graph_mode:
        api.set_timing(plan, True)
        for _ in range(3):
            api.fmm_apply_device(plan, q_dev.data_ptr(), u_dev.data_ptr(), nrhs, sp)
        torch.cuda.synchronize(dev)
    phases = api.get_timings(plan)
    api.set_timing(plan, False)
    if dist:
        tt = torch.tensor([ms_step], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    # points x right-hand sides per second (nrhs = 1 on the headline)
    value = ws * n * nrhs / (ms_step * 1e-3) / 1e6

    u_gpu = u_dev.cpu().numpy()
    if nrhs > 1:
        u_gpu = np.asfortranarray(u_gpu.T)
    u0 = u_gpu if nrhs == 1 else u_gpu[:, 0]
    q0 = q if nrhs == 1 else q[:, 0]

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
    e2e_value = ws * n * nrhs / t_e2e / 1e6
    bytes_col = n * nrhs * (16 if cplx else 8)

    # ---- accuracy vs the dense sum on sampled targets (GPU direct sum) ----
    rng = np.random.default_rng(0xC2B2AE3D27D4EB4F)
    targets = np.sort(rng.choice(n, size=min(args.check_targets, n), replace=False)).astype(np.int32)
    ref_t = api.direct_sum_subset(kern, args.kappa, pts, q0, targets, device=dev)
    relerr_direct = api.max_rel_err(u0[targets], ref_t) if targets.size else None
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
    achieved = w_k2 / (k2_ms * 1e-3) / 1e12
    traffic = pipe = None
    prof = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            key = f"{args.kernel}_{args.dist}_{n}_{args.leaf}_{args.tol}"
            traffic = pj.get(key)
            pipe = pj.get("_fp64_pipe_active", {}).get(key)
        except (OSError, ValueError):
            traffic = pipe = None
    phase_ms = {nm: float(np.mean(phases[:, i])) for i, nm in enumerate(api.PHASES)} if len(phases) else {}
    # interpolation GEMVs: each reads T once per apply
    sb = 16 if cplx else 8
    t_bytes = info.m_proj * sb
    gemv_gbs = {
        "upward": t_bytes / (phase_ms.get("upward", float("nan")) * 1e-3) / 1e9,
        "downward": t_bytes / (phase_ms.get("downward", float("nan")) * 1e-3) / 1e9,
    }

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators: points seed 1, charges seed 1^0x9e3779b97f4a7c15)",
        "config": {
            "workload": f"{args.kernel} {args.dist} N={n:.0e} leaf={args.leaf} tol={args.tol} nrhs={nrhs}",
            "n_points": n, "leaf_cap": args.leaf, "tol": args.tol, "nrhs": nrhs,
            "baseline_config": args.config or "headline (3D Laplace cube N=1e7)",
            "value_definition": "points x right-hand sides per second of device time",
            "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
            "l2": "inputs larger than L2 (resident plan %.1f GB vs 126 MB L2)" % (info.device_bytes / 1e9),
        },
        "roofline": {
            "bound": "fp64", "kernel": "k2_translate (fused ifo/ifs/tfo/level-1)",
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak if fp64_peak > 0 else None,
            "traffic": traffic,
            "fp64_pipe_active": pipe,
            "peak_source": "DFMA loop measured in this run (MEASURED_PEAKS.json has no FP64 figure); nominal 37.2",
            "work": (f"SURVEY.md 8d reference-equivalent: {g_k + 2 * s_c * r_pass:g} flop per dense pair "
                     f"+ {r_pass * 2 * s_c:g} per skeleton pair"),
            "frac_note": ("reference-equivalent work over K2 time can exceed the peak: symmetric "
                          "blocks are generated once and cancelling pairs skipped; fp64_pipe_active "
                          "is the physical FP64 pipe utilisation of the same kernel (ncu, "
                          "profiles/k2_traffic.json)"),
            "p_dense": info.p_dense, "p_skel": info.p_skel, "k2_ms": k2_ms,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bytes_col,
                "d2h_bytes_per_step": bytes_col, "ms_per_step": t_e2e * 1e3,
                "matches_device_result": e2e_same},
        "gpu_launches": int(info.launches_per_apply) * args.steps,
        "clocks": clk,
        "phase_ms": phase_ms,
        "timed_region": ("CUDA graph replay; phase_ms/roofline from 3 extra event-timed applies"
                         if graph_mode else "stream launches with per-phase events in every step"),
        "gemv_gbs": gemv_gbs,
        "relerr_vs_direct": relerr_direct, "n_check": int(targets.size),
        "precompute": {"t_generate_s": t_gen, "t_tree_s": hinfo["t_tree"],
                       "t_skel_s": hinfo["t_skel"], "t_upload_s": t_upload,
                       "depth": hinfo["depth"], "n_boxes": hinfo["n_boxes"],
                       "k_max": hinfo["k_max"], "m_proj": hinfo["proj_scalars"],
                       "host_threads": host.get_threads(),
                       "tree": "GPU tree builder (sfmm_gpu_build_tree)",
                       "skeletons": "GPU skeletonizer (sfmm_gpu_build_skeletons)",
                       "operators": "device-resident, plan built device-to-device "
                       "(sfmm_gpu_plan_create_skel)"},
    }

    # ---- CPU baseline: the unmodified reference apply on the same plan ----
    if rank == 0 and ws == 1 and args.cpu != "off":
        try:
            from oracle import pyoracle as po
            if args.cpu == "full":
                hp.fetch_T()  # the CPU reference needs the operators on the host
                rp = po.RefPipeline.from_desc(hp.desc_struct())
                t0 = time.perf_counter()
                u_ref, _ = rp.apply(q0, cplx)  # the reference apply takes one RHS
                t_cpu = time.perf_counter() - t0
                rp.close()
                out["relerr_vs_cpu_ref"] = po.rel_l2(u0, u_ref)
                out["max_relerr_vs_cpu_ref"] = api.max_rel_err(u0, u_ref)
                n_cpu = n
                sample = (f"full workload (N={n:.0e}), one reference fmm_apply (one RHS) on the "
                          "same tree/skeletons/charges as the GPU run")
            else:
                n_cpu = int(args.ref_n)
                p2 = host.generate_points(args.dist, n_cpu, 1)
                q2 = (host.generate_charges_complex if cplx else host.generate_charges)(
                    n_cpu, 1 ^ CHARGE_STREAM)
                rp = po.RefPipeline.build(kern, p2, args.leaf, args.tol, args.kappa)
                t0 = time.perf_counter()
                rp.apply(q2, cplx)
                t_cpu = time.perf_counter() - t0
                sample = (f"N={n_cpu:.0e} instance of the same workload, one reference fmm_apply "
                          "(one RHS; the reference has no multi-RHS apply)")
            out["cpu_baseline"] = {
                "value": n_cpu / t_cpu / 1e6, "unit": UNIT,
                "cores": po.ref_lib().ref_num_threads(), "kind": "reference",
                "sample": sample, "seconds": t_cpu}
        except Exception as e:  # the checker may be absent; never the product
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None,
                                   "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        emit(out)
    plan.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
