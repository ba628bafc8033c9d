"""B200-native NLINV / IRGNM hot path (arXiv:1301.1215): libnlinv.so + its ctypes binding."""
from .nlinv import NlinvError, Pca, Plan, build_info, coil_partition, get_unique_id, radial_mask  # noqa: F401
