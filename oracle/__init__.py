"""CPU fp64 oracle for the NLINV / IRGNM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product (``paper_1301_1215_b200``
and ``libnlinv.so``) never imports, links or executes it, and it shares no code,
tables or constants generators with the CUDA path.
"""
from .nlinv_oracle import *  # noqa: F401,F403
