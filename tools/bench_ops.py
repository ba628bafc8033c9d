"""BASELINE config 5: operator micro-benchmark against the HBM roofline.

forward / adjoint / normal and the batched 2D FFT for ng in 64..1024 x J in 8..64 coils, on
seeded random operands (splitmix64 U[-1,1), seed 1) and the C2-style radial mask rasterised at
that ng. Median of 50 timed calls after 5 warm-ups, CUDA events on the launching stream.
Algorithmic (compulsory) bytes per call, SURVEY.md §8(d):
  normal  (20 J + 22) N      forward (16 J + 6) N      adjoint (18 J + 14) N
  fft2d   16 J N (one read + one write of each image)
Writes one JSON line per (op, ng, J) and a markdown table to stdout.

python tools/bench_ops.py [--ng 384,1024] [--coils 8,64] [--reps 50]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1301_1215_b200 import NlinvError, Plan, radial_mask  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def timeit(fn, reps, warm=5):
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


def rand_c64(seed, shape):
    n = int(np.prod(shape))
    u = synth.splitmix64_uniform(seed, 2 * n).astype(np.float32)
    return torch.from_numpy(u.view(np.complex64).reshape(shape)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ng", default="64,128,256,384,512,768,1024")
    ap.add_argument("--coils", default="8,16,32,64")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    P = peak()
    rows = []
    for ng in [int(v) for v in args.ng.split(",")]:
        for J in [int(v) for v in args.coils.split(",")]:
            N = ng * ng
            try:
                plan = Plan(ng, J, radial_mask(ng, 15, 5, 0))
            except NlinvError as e:
                print(json.dumps({"ng": ng, "coils": J, "skipped": str(e)}), flush=True)
                continue
            x = rand_c64(1, plan.x_shape)
            dx = rand_c64(2, plan.x_shape)
            dy = rand_c64(3, plan.y_shape)
            y = torch.empty(plan.y_shape, dtype=torch.complex64, device="cuda")
            out = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
            img = rand_c64(4, (J, ng, ng))
            imo = torch.empty_like(img)
            plan.set_point(x)
            ops = {
                "normal": (lambda: plan.normal(0.37, dx, out), (20 * J + 22) * N),
                "forward": (lambda: plan.forward(x, y), (16 * J + 6) * N),
                "adjoint": (lambda: plan.adjoint(dy, out), (18 * J + 14) * N),
                "fft2d": (lambda: plan.fft2d(img, False, imo), 16 * J * N),
            }
            for name, (fn, nbytes) in ops.items():
                ms = timeit(fn, args.reps)
                if name != "fft2d":
                    plan.set_point(x)  # forward() moved the point; keep it fixed
                gbs = nbytes / (ms * 1e-3) / 1e9
                r = {"op": name, "ng": ng, "coils": J, "ms": round(ms, 4), "algorithmic_MB": round(nbytes / 1e6, 2),
                     "GBps": round(gbs, 1), "frac_hbm": round(gbs / P, 3)}
                rows.append(r)
                print(json.dumps(r), flush=True)
            plan.close()
            del x, dx, dy, y, out, img, imo
            torch.cuda.empty_cache()
    print()
    print(f"| op | ng | coils | ms | algorithmic MB | GB/s | frac of {P:.0f} GB/s |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['op']} | {r['ng']} | {r['coils']} | {r['ms']} | {r['algorithmic_MB']} | {r['GBps']} | {r['frac_hbm']} |")


if __name__ == "__main__":
    main()
