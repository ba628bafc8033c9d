"""How many thread-block clusters of the fused K2-K3-K4 kernel can be co-resident (cudaOccupancyMaxActiveClusters)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_1215_b200 as B  # noqa: E402

from paper_1301_1215_b200 import nlinv as N
lib = N._lib
lib.nlinv_debug_k234_clusters.restype = ctypes.c_int
for ng in (192, 256, 384):
    print(ng, "max active clusters:", lib.nlinv_debug_k234_clusters(ng))
