"""PCA channel compression micro-benchmark on one B200.

A C4-shaped frame (32 coils, 384^2 gridded k-space = 147456 samples per channel) compressed to
Jc channels. fit = covariance + Jacobi + sign convention (once per stream); apply = projection of
one frame (per frame). Median of 50 after 5 warm-ups, CUDA events on the launching stream.
Algorithmic bytes: fit reads J N c64 once; apply reads J N and writes Jc N c64.
python tools/bench_pca.py [--coils 32] [--keep 12] [--ng 384]
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
from paper_1301_1215_b200 import Pca  # noqa: E402


def timeit(fn, reps=50, warm=5):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coils", type=int, default=32)
    ap.add_argument("--keep", type=int, default=12)
    ap.add_argument("--ng", type=int, default=384)
    ap.add_argument("--frames", type=int, default=1, help="frames per apply call (batched samples)")
    a = ap.parse_args()
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as fh:
        peak = float(json.load(fh)["hbm_gbs"])
    _, _, y = synth.frame_inputs(a.coils, a.ng)
    Y = torch.from_numpy(np.ascontiguousarray(np.tile(y.astype(np.complex64), (1, a.frames, 1)))).cuda()
    N = Y.numel() // a.coils
    pca = Pca(a.coils, a.keep)
    out = torch.empty((a.keep,) + tuple(Y.shape[1:]), dtype=torch.complex64, device="cuda")
    t_fit = timeit(lambda: pca.fit(Y))
    t_apply = timeit(lambda: pca.apply(Y, out))
    _, w, e, _ = pca.result()
    fb = 8 * a.coils * N
    ab = 8 * (a.coils + a.keep) * N
    print(json.dumps({
        "coils": a.coils, "keep": a.keep, "ng": a.ng, "samples_per_channel": N, "energy_kept": e,
        "fit_ms": round(t_fit, 4), "fit_GBps": round(fb / (t_fit * 1e-3) / 1e9, 1),
        "apply_ms": round(t_apply, 4), "apply_GBps": round(ab / (t_apply * 1e-3) / 1e9, 1),
        "apply_frac_hbm": round(ab / (t_apply * 1e-3) / 1e9 / peak, 3), "peak_GBps": peak,
        "apply_algorithmic_MB": round(ab / 1e6, 2)}))


if __name__ == "__main__":
    main()
