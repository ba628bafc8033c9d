#!/bin/bash
# Box probe: device limits that shape the design, host cores for the CPU baseline.
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm,clocks.max.mem,power.limit --format=csv
nvidia-smi topo -m
echo "nproc: $(nproc)"; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"
python - <<'PY'
import ctypes, torch
p = torch.cuda.get_device_properties(0)
print(p)
rt = ctypes.CDLL("libcudart.so.12") if False else None
import cuda.bindings.runtime as cr
def attr(a):
    err, v = cr.cudaDeviceGetAttribute(a, 0)
    return v
A = cr.cudaDeviceAttr
for name in ("cudaDevAttrMultiProcessorCount", "cudaDevAttrL2CacheSize", "cudaDevAttrMaxSharedMemoryPerBlockOptin",
             "cudaDevAttrMaxSharedMemoryPerMultiprocessor", "cudaDevAttrMaxRegistersPerMultiprocessor",
             "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize",
             "cudaDevAttrClusterLaunch", "cudaDevAttrCooperativeLaunch", "cudaDevAttrMaxBlocksPerMultiprocessor"):
    try:
        print(name, attr(getattr(A, name)))
    except Exception as e:
        print(name, "n/a", e)
PY
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
