// Throughput probe: scalar FFMA vs packed FFMA2 / FADD2 on sm_100a (one launch each, clock64 timing).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void scalar_fma(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  const float b = 1.0001f, c = 0.0001f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void packed_fma(float* out, int iters) {
  u64 a[8];
  for (int i = 0; i < 8; ++i) { float2 f = make_float2(threadIdx.x * 0.001f + i, i + 0.5f); a[i] = *reinterpret_cast<u64*>(&f); }
  float2 bf = make_float2(1.0001f, 1.0001f), cf = make_float2(0.0001f, 0.0001f);
  u64 b = *reinterpret_cast<u64*>(&bf), c = *reinterpret_cast<u64*>(&cf);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&a[i]); s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void packed_add(float* out, int iters) {
  u64 a[8];
  for (int i = 0; i < 8; ++i) { float2 f = make_float2(threadIdx.x * 0.001f + i, i + 0.5f); a[i] = *reinterpret_cast<u64*>(&f); }
  float2 cf = make_float2(0.0001f, 0.0001f);
  u64 c = *reinterpret_cast<u64*>(&cf);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(c));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&a[i]); s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void scalar_add(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  const float c = 0.0001f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c));
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  const int iters = 4096, blocks = 148 * 8, threads = 512;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(float*, int)) {
    k<<<blocks, threads>>>(out, iters); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = (double)blocks * threads * iters * 16;   // 16 float lanes per iteration in every kernel
    printf("%-12s %.3f ms  %.1f T lane-ops/s\n", name, ms, lane_ops / ms / 1e9);
  };
  run("scalar_fma", scalar_fma); run("packed_fma", packed_fma); run("scalar_add", scalar_add); run("packed_add", packed_add);
  return 0;
}
