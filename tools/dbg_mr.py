"""Debug the in-process multi-rank operators step by step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1301_1215_b200 as B
from paper_1301_1215_b200 import radial_mask

mode = sys.argv[1]
ng, J, G = 64, 5, 2
mask = radial_mask(ng, 11, 1, 1)
plans = [B.Plan(ng, J, mask, rank=r, world=G) for r in range(G)]
for p in plans:
    p.connect_local(plans)
streams = [torch.cuda.Stream() for _ in plans]
x = synth.random_complex(31, (J + 1, ng, ng)).astype(np.complex64)
dy = (synth.random_complex(33, (J, ng, ng)) * mask).astype(np.complex64)
xl = [torch.from_numpy(np.ascontiguousarray(np.concatenate([x[:1], x[1 + p.first:1 + p.first + p.count]]))).cuda() for p in plans]
dyl = [torch.from_numpy(np.ascontiguousarray(dy[p.first:p.first + p.count])).cuda() for p in plans]
outs = [torch.empty(p.x_shape, dtype=torch.complex64, device="cuda") for p in plans]
torch.cuda.synchronize()
print("streams", [s.cuda_stream for s in streams], flush=True)
for p, s, a in zip(plans, streams, xl):
    p.set_point(a, stream=s)
torch.cuda.synchronize()
print("set_point ok", flush=True)
t0 = time.time()
for p, s, c, o in zip(plans, streams, dyl, outs):
    p.adjoint(c, o, stream=s)
    print("enqueued adjoint rank", p.rank, time.time() - t0, flush=True)
    if mode == "sync":
        time.sleep(0.5)
torch.cuda.synchronize()
print("adjoint ok", time.time() - t0, flush=True)
dx = synth.random_complex(32, (J + 1, ng, ng)).astype(np.complex64)
dxl = [torch.from_numpy(np.ascontiguousarray(np.concatenate([dx[:1], dx[1 + p.first:1 + p.first + p.count]]))).cuda() for p in plans]
torch.cuda.synchronize()
t0 = time.time()
for p, s, b in zip(plans, streams, dxl):
    p.normal(0.37, b, stream=s)
    print("enqueued normal rank", p.rank, time.time() - t0, flush=True)
torch.cuda.synchronize()
print("normal ok", time.time() - t0, flush=True)
for p, s, a, c, b in zip(plans, streams, xl, dyl, dxl):
    p.set_point(a, stream=s)
    p.adjoint(c, stream=s)
    p.normal(0.37, b, stream=s)
    print("enqueued all rank", p.rank, time.time() - t0, flush=True)
torch.cuda.synchronize()
print("all ok", time.time() - t0, flush=True)
