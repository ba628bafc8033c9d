"""GPU gridding front end at C2: raw radial samples in, image out, per frame.

Times nlinv_stream_frame_radial (pinned host raw samples [12, 15, 384] -> H2D -> GPU gridding ->
7 Newton x 10 CG with the previous frame as prior -> image D2H) for nearest-cell gridding (R20) and
Kaiser-Bessel convolution gridding with the real-valued P_k (R22), plus the gridding kernel alone.
python tools/bench_gridding.py [--frames 40]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1301_1215_b200 import Plan, radial_mask  # noqa: E402

NG, J, S, T = 384, 12, 15, 5


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=40)
    a = ap.parse_args()
    raws = [np.ascontiguousarray(synth.radial_frame_inputs(J, NG, S, T, f, t=f).astype(np.complex64)) for f in range(T)]
    out = {}
    for kernel in ("nearest", "kb"):
        plan = Plan(NG, J, radial_mask(NG, S, T, 0))
        t0 = time.perf_counter()
        plan.set_trajectory(S, T, kernel=kernel, width=4.0)
        setup_s = time.perf_counter() - t0
        hraw = [torch.from_numpy(r).pin_memory() for r in raws]
        himg = torch.empty(plan.image_shape, dtype=torch.complex64).pin_memory()
        draw = torch.from_numpy(raws[0]).cuda()
        y = torch.zeros(plan.y_shape, dtype=torch.complex64, device="cuda")
        st = torch.cuda.current_stream()
        for _ in range(5):
            plan.grid_radial(0, draw, y)
        torch.cuda.synchronize()
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan.grid_radial(0, draw, y)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        plan.stream_reset()
        for i in range(6):
            plan.stream_frame_radial(hraw[i % T], i, 7, 10, himg)
        lat = []
        w0 = time.perf_counter()
        for k in range(a.frames):
            i = 6 + k
            t1 = time.perf_counter()
            plan.stream_frame_radial(hraw[i % T], i, 7, 10, himg)
            lat.append((time.perf_counter() - t1) * 1e3)
        wall = time.perf_counter() - w0
        out[kernel] = {"trajectory_setup_s": round(setup_s, 3), "grid_kernel_ms": round(statistics.median(ts), 4),
                       "e2e_fps": round(a.frames / wall, 2), "latency_ms_p50": round(statistics.median(lat), 3),
                       "latency_ms_max": round(max(lat), 3), "h2d_bytes_per_frame": int(raws[0].nbytes)}
        plan.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
