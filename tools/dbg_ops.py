"""Debug: one operator round (forward/derivative/adjoint/normal) at a given ng, J (single rank)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

ng, J = int(sys.argv[1]), int(sys.argv[2])
mask = radial_mask(ng, 9, 1, 1)
x = torch.from_numpy(synth.random_complex(1, (J + 1, ng, ng)).astype(np.complex64)).cuda()
dy = torch.from_numpy((synth.random_complex(2, (J, ng, ng)) * mask).astype(np.complex64)).cuda()
p = Plan(ng, J, mask)
for name, fn in (("forward", lambda: p.forward(x)), ("derivative", lambda: p.derivative(x)),
                 ("adjoint", lambda: p.adjoint(dy)), ("normal", lambda: p.normal(0.37, x))):
    fn()
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
