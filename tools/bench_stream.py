"""BASELINE config 4 on one B200: a 32-coil 384^2 radial frame stream with previous-frame prior.

SURVEY.md §8(d) C4: ng = 384, J = 32, 15 spokes/frame over T = 5 turns, 7 Newton x 10 CG, 200
frames with the A14 motion (ellipses 3-4 scaled by 1 + 0.1 sin(2 pi t / 25)); the motion period
(25) is a multiple of T, so the 25 distinct synthetic frames are generated once and cycled.
fps = 200 / time after 5 warm-up frames; per-frame latency p50 / p95 / max.

Two measurements, both through libnlinv.so:
  device : nlinv_reconstruct on device-resident frames, CUDA events around every frame
  e2e    : nlinv_stream_frame_compact per frame (pinned host samples at P_k + mask in, image out),
           host wall clock around each call (the call returns after the image is on the host)

python tools/bench_stream.py [--coils 32] [--frames 200] [--warmup 5]
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

PERIOD = 25


def pct(v, q):
    s = sorted(v)
    return s[min(len(s) - 1, int(round(q * (len(s) - 1))))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coils", type=int, default=32)
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ng", type=int, default=384)
    ap.add_argument("--spokes", type=int, default=15)
    ap.add_argument("--turns", type=int, default=5)
    ap.add_argument("--newton", type=int, default=7)
    ap.add_argument("--cg", type=int, default=10)
    ap.add_argument("--compress", type=int, default=0,
                    help="PCA-compress the coils to this many channels on the GPU before each frame (P:241)")
    args = ap.parse_args()
    global NG, SPOKES, TURNS, NEWTON, CG
    NG, SPOKES, TURNS, NEWTON, CG = args.ng, args.spokes, args.turns, args.newton, args.cg
    J = args.coils
    t0 = time.perf_counter()
    frames, masks = [], []
    for f in range(PERIOD):
        _, _, y = synth.frame_inputs(J, NG, t=f)
        frames.append(np.ascontiguousarray(y.astype(np.complex64)))
        masks.append(radial_mask(NG, SPOKES, TURNS, f))
    gen_s = time.perf_counter() - t0

    Jr = args.compress if args.compress else J
    plan = Plan(NG, Jr, masks[0])
    dframes = [torch.from_numpy(f).cuda() for f in frames]
    pca = None
    if args.compress:
        from paper_1301_1215_b200 import Pca
        pca = Pca(J, Jr).fit(dframes[0])          # compression matrix from the first frame
        ycomp = torch.empty((Jr, NG, NG), dtype=torch.complex64, device="cuda")
    dmasks = [torch.from_numpy(m).cuda() for m in masks]
    x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
    img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
    st = torch.cuda.current_stream()

    def frame(i, first):
        plan.set_mask(dmasks[i % PERIOD])
        src = dframes[i % PERIOD]
        if pca is not None:
            src = pca.apply(src, ycomp)
        plan.reconstruct(src, None if first else x, NEWTON, CG, x_out=x, image_out=img)

    frame(0, True)
    for i in range(1, args.warmup + 1):
        frame(i, False)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.frames)]
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(st)
    for k in range(args.frames):
        ev[k][0].record(st)
        frame(args.warmup + 1 + k, False)
        ev[k][1].record(st)
    g1.record(st)
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) for a, b in ev]
    total = g0.elapsed_time(g1)

    if pca is not None:   # the streaming API takes already-compressed samples
        out = {"config": f"C4 (1 GPU) with GPU PCA compression {J} -> {Jr} channels per frame", "coils": J,
               "compressed_to": Jr, "energy_kept": pca.result()[2], "frames": args.frames,
               "device": {"fps": round(args.frames / (total / 1e3), 2), "latency_ms_p50": round(pct(lat, 0.5), 4),
                          "latency_ms_p95": round(pct(lat, 0.95), 4), "latency_ms_max": round(max(lat), 4)}}
        print(json.dumps(out))
        return
    # end to end through the public streaming API, one frame at a time
    hs = [torch.from_numpy(np.ascontiguousarray(f.reshape(J, -1)[:, np.flatnonzero(m)])).pin_memory()
          for f, m in zip(frames, masks)]
    hm = [torch.from_numpy(m).pin_memory() for m in masks]
    himg = torch.empty(plan.image_shape, dtype=torch.complex64).pin_memory()
    plan.stream_reset()
    for i in range(args.warmup + 1):
        plan.stream_frame_compact(hs[i % PERIOD], hm[i % PERIOD], NEWTON, CG, himg)
    e2e = []
    w0 = time.perf_counter()
    for k in range(args.frames):
        i = args.warmup + 1 + k
        a = time.perf_counter()
        plan.stream_frame_compact(hs[i % PERIOD], hm[i % PERIOD], NEWTON, CG, himg)
        e2e.append((time.perf_counter() - a) * 1e3)
    wall = time.perf_counter() - w0
    out = {
        "config": "C4 (1 GPU)" if (NG, J) == (384, 32) else "custom", "ng": NG, "coils": J, "spokes": SPOKES, "turns": TURNS, "newton": NEWTON, "cg": CG,
        "frames": args.frames, "warmup": args.warmup, "distinct_frames": PERIOD,
        "device": {"fps": round(args.frames / (total / 1e3), 2), "latency_ms_p50": round(pct(lat, 0.5), 4),
                   "latency_ms_p95": round(pct(lat, 0.95), 4), "latency_ms_max": round(max(lat), 4),
                   "latency_ms_mean": round(statistics.mean(lat), 4)},
        "e2e": {"fps": round(args.frames / wall, 2), "latency_ms_p50": round(pct(e2e, 0.5), 4),
                "latency_ms_p95": round(pct(e2e, 0.95), 4), "latency_ms_max": round(max(e2e), 4),
                "h2d_bytes_per_frame": int(max(h.numel() for h in hs) * 8 + masks[0].nbytes),
                "d2h_bytes_per_frame": int(himg.numel() * 8)},
        "input_generation_s": round(gen_s, 1),
    }
    print(json.dumps(out))
    plan.close()


if __name__ == "__main__":
    main()
