"""Build libnlinv.so (sm_100a) in-tree with nvcc: one object per grid size, compiled in parallel."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libnlinv.so")
SIZES = (16, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401  (torch's own NCCL 2.28; one libnccl per process)
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except Exception:
        pass
    return None, None


def _sources_digest(extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for f in sorted(glob.glob(os.path.join(CSRC, "*"))) + [os.path.join(INCLUDE, "nlinv.h"), __file__]:
        with open(f, "rb") as fh:
            h.update(f.encode())
            h.update(fh.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "nvcc")
    nccl_inc, nccl_lib = _nccl_dirs()
    defs = ["-DNLINV_WITH_NCCL", "-I" + nccl_inc] if nccl_inc else []
    defs += [d for d in os.environ.get("NLINV_DEFS", "").split() if d]
    digest = _sources_digest(" ".join(defs))
    stamp = LIB + ".sha256"
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == digest:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    for L in SIZES:
        jobs.append(([nvcc, *ARCH, *FLAGS, *defs, f"-DNLV_L={L}", "-c", os.path.join(CSRC, "inst.cu"),
                      "-o", os.path.join(OBJ, f"inst_{L}.o")], f"inst_{L}"))
    for name in ("nlinv_kernels", "nlinv_capi", "pca"):
        jobs.append(([nvcc, *ARCH, *FLAGS, *defs, "-c", os.path.join(CSRC, name + ".cu"),
                      "-o", os.path.join(OBJ, name + ".o")], name))

    def run(job):
        cmd, name = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(f"[build] {name} ok\n")
        return name

    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, f"inst_{L}.o") for L in SIZES] + [os.path.join(OBJ, n + ".o")
                                                                 for n in ("nlinv_kernels", "nlinv_capi", "pca")]
    link = [nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs]
    if nccl_lib:
        link += ["-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_lib]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(link)}\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as fh:
        fh.write(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
