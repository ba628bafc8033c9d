#!/usr/bin/env python
"""NLINV frame-rate benchmark (BASELINE.json metric) through libnlinv.so's C ABI.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
For N > 1 launch with torch.distributed.run (one rank per GPU); coils are sharded over ranks
(strong scaling, BASELINE config 3).

A step = one full NLINV frame of BASELINE config 2: 12 coils, 384^2 grid (192^2 image), 15 radial
spokes rotated over 5 turns, 7 Newton x 10 CG, the previous frame's x as prior.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

NG, J, SPOKES, TURNS, NEWTON, CG = 384, 12, 15, 5, 7, 10
METRIC = "NLINV frames/sec and per-frame latency at 1/2/4/8 B200; % HBM roofline"
WORKLOAD = ("C2: 12-coil 192x192 image on a 2x oversampled 384x384 grid, 15 radial spokes/frame "
            "(5 turns), 7 Newton x 10 CG, frame stream with previous-frame prior")


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# Algorithmic (compulsory) bytes per launch, each operand read once and each result written once
# at its minimal support (DESIGN.md §7 Roofline). N = ng^2, Jl = local coils, c64 = 8 B.
def algo_bytes(name: str, ng: int, Jl: int, L: int = CG) -> float:
    N = ng * ng
    t = {
        # K1: r, p, dx in; p, dx, T1 out per coil (+ rho slice, w^-1); dx skipped at iterations 0-1
        "col_ifft_w_cg": (8 + 8 + 8 + 8 + 8 + 4) * Jl * N + 4 * N + 40 * N,
        "row_k2": 10 * Jl * N + 4 * N,
        "col_psf": 8 * Jl * N + N,
        "row_k4": 10 * Jl * N + 4 * N,
        "col_fft_w_normal": 20 * Jl * N + 4 * N + 18 * N,   # + rho slice: S, p_rho in, Ap_rho out
        # K5 fused with the CG update and K1 of the next iteration on the same tile. Compulsory operands only, each
        # counted once per launch: per coil T4 (Omega rows) 4, p 8, r 8+8, dx 8+8, p out 8, T1 out 4;
        # w^-1 once; rho block: coil-sum plane 2, p 8, r 8+8, dx 8+8, p out 8 (the A p_rho round
        # trip and the second p read are implementation re-reads, not counted)
        "col_k5_cg_k1": 56 * Jl * N + 4 * N + 50 * N,
        # ... last iteration: + the Newton update x += dx + gamma p (T4, p, dx, x in; x out)
        "col_k5_newton": 36 * Jl * N + 4 * N + 34 * N,
        # Newton rhs + K1 of CG iteration 0 (T1 out)
        # T in 4, chat 8, chat_ref 8, b out once 8 (r = p = b), T1 out 4; w^-1; rho block
        "col_rhs_k1": 32 * Jl * N + 4 * N + 34 * N,
        "r_update": 24 * N * (Jl + 1),                       # r, Ap in; r out
        "newton_update": 32 * N * (Jl + 1),                  # p, dx, x in; x out
        "col_ifft_w": 8 * Jl * N + 4 * N + 4 * Jl * N,
        "row_setpoint_fwd": 4 * Jl * N + 2 * Jl * N + 4 * Jl * N + 2 * N + 2 * N,
        "row_setpoint": 4 * Jl * N + 2 * Jl * N + 4 * N,
        "row_rss": 4 * Jl * N + 2 * Jl * N + 4 * N + 1 * N,
        "col_resadj": 4 * Jl * N + 8 * Jl * N + N + 4 * Jl * N,
        "col_fft_w_rhs": 4 * Jl * N + 8 * Jl * N + 8 * Jl * N + 4 * N + 16 * Jl * N + 34 * N,
        "init_x": 8 * N * (Jl + 1),
        "image": 2 * N + N + 2 * N,
    }
    return float(t.get(name, 0.0))


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(device)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_frames(rank_first: int, count: int):
    """T distinct synthetic frames (moving phantom, rotated spokes) for this rank's coils."""
    import synth
    from paper_1301_1215_b200 import radial_mask
    frames, masks = [], []
    for f in range(TURNS):
        _, _, y = synth.frame_inputs(J, NG, t=f)
        frames.append(np.ascontiguousarray(y[rank_first:rank_first + count].astype(np.complex64)))
        masks.append(radial_mask(NG, SPOKES, TURNS, f))
    return frames, masks


def run_ours(args):
    import torch
    if os.environ.get("NLINV_BENCH_STREAM") == "1":
        torch.cuda.set_device(_dist()[2])
        with torch.cuda.stream(torch.cuda.Stream()):
            return _run_ours(args)
    return _run_ours(args)


def _run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1301_1215_b200 import Plan

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1301_1215_b200 import radial_mask
    from paper_1301_1215_b200.dist import connect_peers, exchange_unique_id
    mask0 = radial_mask(NG, SPOKES, TURNS, 0)
    if world > 1 and args.transport == "nccl":
        plan = Plan(NG, J, mask0, rank=rank, world=world, nccl_id=exchange_unique_id(rank, world))
    else:
        # peer-memory exchange (default): every rank maps every rank's exchange window (CUDA IPC)
        plan = Plan(NG, J, mask0, rank=rank, world=world)
        if world > 1:
            connect_peers(plan)
    frames, masks = make_frames(plan.first, plan.count)
    dframes = [torch.from_numpy(f).cuda() for f in frames]
    dmasks = [torch.from_numpy(m).cuda() for m in masks]
    frame_dev = torch.empty_like(dframes[0])
    x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
    img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def step(i, first):
        frame_dev.copy_(dframes[i % TURNS])
        plan.set_mask(dmasks[i % TURNS])
        plan.reconstruct(frame_dev, None if first else x, NEWTON, CG, x_out=x, image_out=img)

    # clocks are sampled from the start of warm-up through the end of the timed region
    clocks = Clocks(local)
    time.sleep(0.3)
    # warm-up (also captures the CUDA graph of the warm-frame configuration)
    step(0, True)
    for i in range(max(args.warmup, 3)):
        step(i + 1, False)
    torch.cuda.synchronize()
    barrier()

    # timed region: K frames, L2 flushed before each, device time from CUDA events on the stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = plan.launch_count
    torch.cuda.synchronize()
    barrier()
    for k in range(args.steps):
        i = args.warmup + 1 + k
        frame_dev.copy_(dframes[i % TURNS])
        flush.zero_()
        ev[k][0].record(stream)
        plan.set_mask(dmasks[i % TURNS])
        plan.reconstruct(frame_dev, x, NEWTON, CG, x_out=x, image_out=img)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    clk["window"] = "warm-up + timed region"
    launches = plan.launch_count - launches0
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(ms_steps)
    if world > 1:
        t = torch.tensor([total_ms] + ms_steps, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0].item())
        ms_steps = [float(v) for v in t[1:].tolist()]   # per-frame latency: the slowest rank
    lat = sorted(ms_steps)

    def pct(q):
        return lat[min(len(lat) - 1, int(round(q * (len(lat) - 1))))]
    fps = args.steps / (total_ms / 1e3)

    # end to end through the public streaming API, every step: the frame's RAW radial samples
    # (pinned host [coils, spokes, ng], exact non-Cartesian acquisition of the phantom) in, GPU
    # gridding (R20, replacing the paper's CPU pre-processing step), reconstruction with the
    # previous frame as prior, image out (nlinv_stream_frame_radial)
    import synth
    plan.set_trajectory(SPOKES, TURNS)
    hraw = [torch.from_numpy(np.ascontiguousarray(
        synth.radial_frame_inputs(J, NG, SPOKES, TURNS, f, t=f)[plan.first:plan.first + plan.count]
        .astype(np.complex64))).pin_memory() for f in range(TURNS)]
    himg = torch.empty(plan.image_shape, dtype=torch.complex64).pin_memory()
    plan.stream_reset()
    for i in range(max(args.warmup, 3) + 1):
        plan.stream_frame_radial(hraw[i % TURNS], i, NEWTON, CG, himg)
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        i = max(args.warmup, 3) + 1 + k
        plan.stream_frame_radial(hraw[i % TURNS], i, NEWTON, CG, himg)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = hraw[0].numel() * 8
    d2h = himg.numel() * 8

    # the same through the compact-frame entry (gridded samples at the cells of P_k, ascending
    # index order, + the mask; the zeros of the full grid never cross PCIe, R18)
    hsamp = [torch.from_numpy(np.ascontiguousarray(f.reshape(f.shape[0], -1)[:, np.flatnonzero(m)])).pin_memory()
             for f, m in zip(frames, masks)]
    hmasks = [torch.from_numpy(m).pin_memory() for m in masks]
    plan.stream_reset()
    for i in range(max(args.warmup, 3) + 1):
        plan.stream_frame_compact(hsamp[i % TURNS], hmasks[i % TURNS], NEWTON, CG, himg)
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        i = k + 1
        plan.stream_frame_compact(hsamp[i % TURNS], hmasks[i % TURNS], NEWTON, CG, himg)
    e2c_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2c_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2c_s = float(t.item())
    h2d_c = max(h.numel() for h in hsamp) * 8 + masks[0].nbytes

    # roofline: one profiled frame (every kernel bracketed by CUDA events on its stream)
    plan.set_profiling(True)
    step(args.warmup + 1 + args.steps, False)
    prof = plan.profile()
    plan.set_profiling(False)
    peak, peak_src = _peaks()
    frame_ms = sum(v["ms"] for v in prof.values())
    top = max(prof.items(), key=lambda kv: kv[1]["ms"])
    tname, tv = top
    tb = algo_bytes(tname, NG, plan.count) * tv["launches"]
    achieved = tb / (tv["ms"] / 1e3) / 1e9
    traffic = ncu_ms = ncu_ms_warm = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(tname, {}).get("dram_bytes_per_launch")
        us = tr.get(tname, {}).get("avg_us_ncu")
        ncu_ms = us / 1e3 if us else None
        usw = tr.get(tname, {}).get("avg_us_ncu_warm")
        ncu_ms_warm = usw / 1e3 if usw else None
    except Exception:
        traffic = ncu_ms = ncu_ms_warm = None
    frame_bytes = sum(algo_bytes(k, NG, plan.count) * v["launches"] for k, v in prof.items())
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 4),
                   "share": round(v["ms"] / frame_ms, 4),
                   "GBps": round(algo_bytes(k, NG, plan.count) * v["launches"] / (v["ms"] / 1e3) / 1e9, 1)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (modified Shepp-Logan + Gaussian coil maps, rasterised radial spokes)",
            "config": {"workload": WORKLOAD, "ng": NG, "coils": J, "spokes": SPOKES, "turns": TURNS,
                       "newton_steps": NEWTON, "cg_iters": CG, "coils_per_rank": plan.count,
                       "parallelism": (f"coil-sharded x{world} ({args.transport} exchange)" if world > 1
                                       else "single GPU"),
                       "l2": "flushed (256 MB write) before every timed frame, outside the events",
                       "per_frame_ms": [round(m, 4) for m in ms_steps]},
            "e2e": {"value": round(args.steps / e2e_s, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "nlinv_stream_frame_radial (pinned host raw radial samples in, GPU gridding, image out)"},
            "e2e_compact": {"value": round(args.steps / e2c_s, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d_c,
                            "d2h_bytes_per_step": d2h,
                            "api": "nlinv_stream_frame_compact (pinned host gridded samples at P_k + mask in, image out)"},
            "latency_ms": {"p50": round(pct(0.5), 4), "p95": round(pct(0.95), 4), "max": round(lat[-1], 4),
                           "what": "device time of one frame (CUDA events around reconstruct), max over ranks"},
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": {"bound": "hbm", "kernel": tname, "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": tb / tv["launches"],
                         "avg_launch_ms": tv["ms"] / tv["launches"],
                         "ncu_avg_launch_ms": ncu_ms,
                         "frac_ncu": (round(tb / tv["launches"] / (ncu_ms / 1e3) / 1e9 / peak, 4) if ncu_ms else None),
                         "ncu_avg_launch_ms_warm": ncu_ms_warm,
                         "frac_ncu_warm": (round(tb / tv["launches"] / (ncu_ms_warm / 1e3) / 1e9 / peak, 4)
                                           if ncu_ms_warm else None),
                         "ncu_note": ("profiles/ncu_traffic.json: ncu launch list of one eager C2 frame, serialised; "
                                      "cold = L2 flushed before every kernel, warm = --cache-control none (the L2 "
                                      "state a frame really sees)"),
                         "share_of_frame": round(tv["ms"] / frame_ms, 4),
                         "frame_algorithmic_GBps": round(frame_bytes / (frame_ms / 1e3) / 1e9, 1),
                         "method": "one extra frame with every kernel bracketed by CUDA events (no graph)",
                         "kernels": kernels},
        }
    plan.close()
    return out, world, rank


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_inputs():
    import oracle as O
    import synth
    _, _, y = synth.frame_inputs(J, NG, t=0)
    y = y.astype(np.complex64).astype(np.complex128)
    P = O.radial_mask(NG, SPOKES, TURNS, 0).astype(np.float64)
    return O, y, P, O.weights_inv(NG), O.fov_mask(NG), O.initial_x(J, NG)


def oracle_time(newton_steps, cores):
    """The fp64 oracle (as it stands) on the C2 workload's frame 0: `newton_steps` IRGNM steps of
    10 CG from the cold start, timed on `cores` host threads (cores > 1: the coil-parallel mode,
    oracle.set_workers, bit-identical results). Returns seconds."""
    O, y, P, winv, M, x0 = _oracle_inputs()
    from threadpoolctl import threadpool_limits
    O.set_workers(cores)
    try:
        with threadpool_limits(limits=1):
            x = x0
            t0 = time.perf_counter()
            for n in range(newton_steps):
                x, _ = O.newton_step(x, x0, y, P, winv, M, 1.0 * (1.0 / 3.0) ** n, CG)
            return time.perf_counter() - t0
    finally:
        O.set_workers(1)


def run_reference(args):
    """--impl reference: the oracle as it stands on all host cores (coil-parallel mode), same metric
    and workload. One step = one IRGNM Newton step (10 CG) of the C2 frame, i.e. 1/7 of a frame:
    the frame rate is steps / 7 / time, and ms_per_step is the measured time of one such step."""
    world, rank, _ = _dist()
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_time(1, cores)
    ts = [oracle_time(1, cores) for _ in range(args.steps)]
    step_s = statistics.mean(ts)
    fps = 1.0 / (NEWTON * step_s)
    sample = (f"one Newton step (10 CG) of the C2 frame per step = 1/{NEWTON} frame; "
              f"{args.steps} timed steps, mean {step_s:.3f} s, on {cores} threads ({_cpu_model()})")
    return {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "ng": NG, "coils": J, "step": f"1/{NEWTON} frame (one Newton step)"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu": _cpu_model()},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _relaunch(args):
    """--gpus N > 1 without a torch.distributed launcher: re-exec this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU exchange: peer memory fused into the kernels (default) or NCCL all-reduces")
    ap.add_argument("--dry-run", action="store_true", help="check the rank launch only (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(_relaunch(args))
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.dry_run:   # launcher check without a GPU: every rank reports over gloo, rank 0 prints
        import torch.distributed as dist
        world, rank, _ = _dist()
        from paper_1301_1215_b200 import coil_partition
        parts = [coil_partition(J, world, r) for r in range(world)]
        if world > 1:
            dist.init_process_group("gloo")
            got = [None] * world
            dist.all_gather_object(got, rank)
            dist.destroy_process_group()
        else:
            got = [0]
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": got, "coils_per_rank": [c for _, c in parts],
                              "transport": args.transport}))
        return
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out))
        return
    out, world, rank = run_ours(args)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            # one whole C2 frame (7 Newton x 10 CG) of the oracle on all host cores (coil-parallel
            # mode), and the same frame on one core
            cores = os.cpu_count() or 1
            t_all = oracle_time(NEWTON, cores)
            t_one = oracle_time(NEWTON, 1) if cores > 1 else t_all
            out["cpu_baseline"] = {"value": round(1.0 / t_all, 6), "unit": "frames/s", "cores": cores, "kind": "oracle",
                                   "cpu": _cpu_model(),
                                   "sample": f"one whole C2 frame (frame 0, 7 Newton x 10 CG, cold start) in "
                                             f"{t_all:.2f} s on {cores} threads (coil-parallel mode)",
                                   "single_core": {"value": round(1.0 / t_one, 6), "unit": "frames/s", "cores": 1,
                                                   "sample": f"the same frame in {t_one:.2f} s on one core"}}
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
