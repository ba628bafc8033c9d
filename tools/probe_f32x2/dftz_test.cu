// DFTZ<4, 0b1001> packed (fp32x2) vs a plain-C reference on one thread
#include <cstdio>
#include "../../paper_1301_1215_b200/csrc/fft.cuh"
using namespace nlv;
template <int DIR, unsigned ZM>
__global__ void k(const float2* in, float2* out) {
  float2 a[4];
  for (int i = 0; i < 4; ++i) a[i] = ((ZM >> i) & 1u) ? make_float2(0.f, 0.f) : in[i];
  DFTZ<4, DIR, ZM>::run(a);
  for (int i = 0; i < 4; ++i) out[i] = a[i];
  float2 b[4];
  for (int i = 0; i < 4; ++i) b[i] = ((ZM >> i) & 1u) ? make_float2(0.f, 0.f) : in[i];
  DFT<4, DIR>::run(b);
  for (int i = 0; i < 4; ++i) out[4 + i] = b[i];
}
int main() {
  float2 h[4] = {{1.f, 2.f}, {3.f, -1.f}, {0.5f, 0.25f}, {-2.f, 4.f}};
  float2 *d, *o; cudaMalloc(&d, 64); cudaMalloc(&o, 128);
  cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  float2 r[8];
  k<-1, 9u><<<1, 1>>>(d, o); cudaMemcpy(r, o, 64, cudaMemcpyDeviceToHost);
  printf("DIR-1 ZM9 dftz:"); for (int i = 0; i < 4; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n      dft:  "); for (int i = 4; i < 8; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n");
  k<1, 9u><<<1, 1>>>(d, o); cudaMemcpy(r, o, 64, cudaMemcpyDeviceToHost);
  printf("DIR+1 ZM9 dftz:"); for (int i = 0; i < 4; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n      dft:  "); for (int i = 4; i < 8; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n");
  k<-1, 6u><<<1, 1>>>(d, o); cudaMemcpy(r, o, 64, cudaMemcpyDeviceToHost);
  printf("DIR-1 ZM6 dftz:"); for (int i = 0; i < 4; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n      dft:  "); for (int i = 4; i < 8; ++i) printf(" (%g,%g)", r[i].x, r[i].y); printf("\n");
  return 0;
}
