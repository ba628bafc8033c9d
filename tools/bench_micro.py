"""the paper's §2.6 micro-benchmarks on B200 + NVLink.

  * batched 2D FFT strong scaling: a fixed batch of ng^2 images split over the ranks, each rank
    transforming its share with libnlinv's centred 2D FFT (nlinv_debug_fft2d); time = max over
    ranks of CUDA-event time; reported as images/s and GB/s (one read + one write per image)
  * axpy strong scaling (the paper's Fig. 4): y = a x + y over a fixed vector of 2^28
    floats split over the ranks (libnlinv's float4 kernel, nlinv_debug_axpy); time = max over ranks;
    GB/s counts 12 bytes per element (x, y read; y written)
  * collective transfer curves: torch.distributed (NCCL) all-reduce and broadcast of 8 B .. 64 MB
    float buffers, median of 20 after 5 warm-ups, bus bandwidth per NCCL's convention

python tools/bench_micro.py                                  # 1 GPU
python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/bench_micro.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1301_1215_b200 import Plan, radial_mask  # noqa: E402
from paper_1301_1215_b200.nlinv import axpy  # noqa: E402


def ev_time(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def maxr(v, world):
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = {"world": world, "fft": [], "axpy": [], "allreduce": [], "broadcast": []}
    for n_total in (1 << 24, 1 << 28):
        share = ((n_total + world - 1) // world + 3) // 4 * 4
        xv = torch.ones(share, dtype=torch.float32, device="cuda")
        yv = torch.zeros(share, dtype=torch.float32, device="cuda")
        ms = maxr(ev_time(lambda: axpy(0.5, xv, yv)), world)
        out["axpy"].append({"n": n_total, "per_rank": share, "ms": round(ms, 4),
                            "GBps_total": round(12.0 * n_total / (ms * 1e-3) / 1e9, 1)})
        del xv, yv
    for ng, batch in ((384, 96), (1024, 32)):
        share = (batch + world - 1) // world
        plan = Plan(ng, 1, radial_mask(ng, 4, 1, 0))
        x = torch.randn(share, ng, ng, dtype=torch.complex64, device="cuda")
        y = torch.empty_like(x)
        ms = maxr(ev_time(lambda: plan.fft2d(x, False, y)), world)
        out["fft"].append({"ng": ng, "batch": batch, "per_rank": share, "ms": round(ms, 4),
                           "images_per_s": round(batch / (ms * 1e-3), 1),
                           "GBps_total": round(16.0 * batch * ng * ng / (ms * 1e-3) / 1e9, 1)})
        plan.close()
    for nbytes in (8, 2048, 295 * 1024, 1 << 20, 16 << 20, 64 << 20):
        n = max(1, nbytes // 4)
        buf = torch.ones(n, dtype=torch.float32, device="cuda")
        if world > 1:
            ar = ev_time(lambda: dist.all_reduce(buf))
            bc = ev_time(lambda: dist.broadcast(buf, 0))
        else:
            ar = bc = 0.0
        ar, bc = maxr(ar, world), maxr(bc, world)
        f = 2.0 * (world - 1) / world
        out["allreduce"].append({"bytes": n * 4, "us": round(ar * 1e3, 2),
                                 "busbw_GBps": round(f * n * 4 / (ar * 1e-3) / 1e9, 1) if ar > 0 else None})
        out["broadcast"].append({"bytes": n * 4, "us": round(bc * 1e3, 2),
                                 "busbw_GBps": round(n * 4 / (bc * 1e-3) / 1e9, 1) if bc > 0 else None})
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
