import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O, synth
import paper_1301_1215_b200 as B
from test_gpu_multirank import make_ranks, c64
variant = sys.argv[1]
ng, J, G = 64, 5, 2
mask = O.radial_mask(ng, 11, 1, 1)
x = c64(synth.random_complex(31, (J + 1, ng, ng)))
dx = c64(synth.random_complex(32, (J + 1, ng, ng)))
dy = c64(synth.random_complex(33, (J, ng, ng)) * mask)
plans = make_ranks(B, ng, J, G, mask)
streams = [torch.cuda.Stream() for _ in plans]
def local(a, p, blocks):
    if blocks == "x":
        return torch.from_numpy(np.ascontiguousarray(np.concatenate([a[:1], a[1 + p.first:1 + p.first + p.count]]))).cuda()
    return torch.from_numpy(np.ascontiguousarray(a[p.first:p.first + p.count])).cuda()
xl = [local(x, p, "x") for p in plans]
dxl = [local(dx, p, "x") for p in plans]
dyl = [local(dy, p, "y") for p in plans]
torch.cuda.synchronize()
t0 = time.time()
for p, s, a, b, c in zip(plans, streams, xl, dxl, dyl):
    p.set_point(a, stream=s); print("sp", p.rank, time.time()-t0, flush=True)
    if variant != "noadj":
        p.adjoint(c, stream=s); print("adj", p.rank, time.time()-t0, flush=True)
    if variant != "nonormal":
        p.normal(0.37, b, stream=s); print("nrm", p.rank, time.time()-t0, flush=True)
torch.cuda.synchronize()
print("ok", time.time()-t0, flush=True)
