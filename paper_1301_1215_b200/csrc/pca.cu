// PCA channel compression on the GPU.
//
// PAPER.md P:241 (§3.2): "A principal component analysis preprocessing step is applied before
// reconstruction to compress the 32 channels to 8-12" [Huang 2007]; J x J
// channel covariance from the data samples, eigendecomposition, projection onto the top-J'
// eigenvectors (descending eigenvalues; sign convention: the largest-magnitude component of each
// eigenvector real-positive).
//
//   C[a][b] = sum_n y_a[n] conj(y_b[n])   cov_partial_kernel (grid-stride tiles, fp64 FMAs from an
//                                          fp64 shared tile, per-CTA partials) + cov_finish_kernel
//                                          (partials summed in CTA order: deterministic)
//   C = V diag(lambda) V^H               jacobi_kernel: one CTA, parallel cyclic complex Jacobi in
//                                          fp64 (round-robin pairing, J/2 disjoint rotations per
//                                          step), then descending sort and the sign convention
//   y'_k[n] = sum_j conj(V[j][k]) y_j[n] pca_apply_kernel: two samples per thread, coalesced
//                                          channel rows, V in shared memory (J reads and J' writes
//                                          of 8 B per sample against J J' complex FMAs)
// The covariance is a J x J x nsamp contraction (0.6 GFLOP for 32 coils on the 384^2 grid) fed by
// one HBM pass over the data and run once per stream (the matrix is then applied to every frame),
// so it uses register-blocked fp32 FMAs with fp64 accumulation across tiles rather than tensor
// cores (TF32 inputs would cost the eigenvector accuracy the parity needs).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/nlinv.h"
#include "nlinv_kernels.cuh"

namespace nlv {
void set_lib_error(const std::string& msg);  // nlinv_capi.cu

namespace {

constexpr int kPcaMaxJ = 32;   // the scanner records up to 32 channels
constexpr int kCovTN = 32;          // samples per shared tile
constexpr int kCovThreads = 256;
constexpr int kCovMaxBlocks = 592;  // 4 x 148 SMs

struct dcplx {
  double x, y;
};

// ---------------------------------------------------------------- covariance
// Register-blocked Gram matrix: thread (group g, block tri) owns the 4 x 4 channel block
// (4 ba.., 4 bb..), ba <= bb, and the samples s = g, g + G, .. of every shared tile, so each
// pair of 4-channel loads feeds 16 complex FMAs. fp32 FMAs inside a tile of kCovTN samples,
// fp64 accumulation across tiles; the G groups are summed in group order in shared memory and
// each CTA writes its partial C blocks; cov_finish_kernel sums the partials in CTA order.
__global__ void __launch_bounds__(kCovThreads) cov_partial_kernel(const float2* __restrict__ Y, int J, long long nsamp,
                                                                 double* __restrict__ part) {
  __shared__ float2 tile[kPcaMaxJ][kCovTN + 1];
  __shared__ double cacc[(kPcaMaxJ / 4) * (kPcaMaxJ / 4 + 1) / 2 * 16 * 2];
  const int J4 = (J + 3) / 4, ntri = J4 * (J4 + 1) / 2;
  const int G = (kCovThreads / ntri) > 0 ? kCovThreads / ntri : 1;
  const int tid = threadIdx.x;
  const bool active = tid < G * ntri;
  const int g = active ? tid / ntri : 0, tri = active ? tid % ntri : 0;
  int ba = 0, rem = tri;
  while (rem >= J4 - ba) {
    rem -= J4 - ba;
    ++ba;
  }
  const int bb = ba + rem;
  double ax[16], ay[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) ax[u] = ay[u] = 0.0;
  const long long ntile = (nsamp + kCovTN - 1) / kCovTN;
  for (long long tt = blockIdx.x; tt < ntile; tt += gridDim.x) {
    const long long n0 = tt * kCovTN;
    __syncthreads();
    for (int i = tid; i < J4 * 4 * kCovTN; i += blockDim.x) {
      const int j = i / kCovTN, sidx = i % kCovTN;
      const long long n = n0 + sidx;
      tile[j][sidx] = (j < J && n < nsamp) ? Y[(size_t)j * nsamp + n] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    if (active) {
      float fx[16], fy[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) fx[u] = fy[u] = 0.f;
      for (int sidx = g; sidx < kCovTN; sidx += G) {
        float2 ya[4], yb[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          ya[i2] = tile[4 * ba + i2][sidx];
          yb[i2] = tile[4 * bb + i2][sidx];
        }
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {   // y_a conj(y_b)
            fx[i2 * 4 + k2] = fmaf(ya[i2].x, yb[k2].x, fmaf(ya[i2].y, yb[k2].y, fx[i2 * 4 + k2]));
            fy[i2 * 4 + k2] = fmaf(ya[i2].y, yb[k2].x, fmaf(-ya[i2].x, yb[k2].y, fy[i2 * 4 + k2]));
          }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        ax[u] += (double)fx[u];
        ay[u] += (double)fy[u];
      }
    }
  }
  // groups summed in group order
  for (int gg = 0; gg < G; ++gg) {
    __syncthreads();
    if (active && g == gg) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        double* c = cacc + ((size_t)tri * 16 + u) * 2;
        c[0] = (gg == 0) ? ax[u] : c[0] + ax[u];
        c[1] = (gg == 0) ? ay[u] : c[1] + ay[u];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < ntri * 32; i += blockDim.x) part[(size_t)blockIdx.x * ntri * 32 + i] = cacc[i];
}

// C (full Hermitian, [J][J] (re, im) fp64) = sum over CTAs in CTA order
__global__ void cov_finish_kernel(const double* __restrict__ part, int nblk, int J, double* __restrict__ C) {
  const int J4 = (J + 3) / 4, ntri = J4 * (J4 + 1) / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ntri * 16; e += gridDim.x * blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int b = 0; b < nblk; ++b) {
      sx += part[((size_t)b * ntri * 16 + e) * 2];
      sy += part[((size_t)b * ntri * 16 + e) * 2 + 1];
    }
    const int tri = e / 16, u = e % 16;
    int ba = 0, rem = tri;
    while (rem >= J4 - ba) {
      rem -= J4 - ba;
      ++ba;
    }
    const int bb = ba + rem;
    const int a = 4 * ba + u / 4, b = 4 * bb + u % 4;
    if (a >= J || b >= J || (ba == bb && a > b)) continue;
    C[(a * J + b) * 2] = sx;
    C[(a * J + b) * 2 + 1] = (a == b) ? 0.0 : sy;
    C[(b * J + a) * 2] = sx;
    C[(b * J + a) * 2 + 1] = (a == b) ? 0.0 : -sy;
  }
}

// ---------------------------------------------------------------- eigendecomposition
// Parallel cyclic Jacobi for the Hermitian C: per step the round-robin schedule pairs every
// index with exactly one other (J even; odd J gets a dummy index), the J/2 rotations are formed
// from the current matrix and applied together (they act on disjoint row/column pairs).
// Rotation of (p, q) with b = A_pq = |b| e^{i phi}: G = D R, D = diag(1, e^{-i phi}),
// R = [[c, s], [-s, c]], t = sgn(tau) / (|tau| + sqrt(1 + tau^2)), tau = (A_qq - A_pp) / (2|b|),
// c = 1 / sqrt(1 + t^2), s = t c; A <- G^H A G zeroes A_pq; V <- V G accumulates eigenvectors.
__global__ void __launch_bounds__(256) jacobi_kernel(const double* __restrict__ Cin, int J, int Jc, float2* __restrict__ Vout,
                                                     double* __restrict__ eig_out, double* __restrict__ energy_out,
                                                     int* __restrict__ sweeps_out) {
  __shared__ dcplx A[kPcaMaxJ][kPcaMaxJ + 1];
  __shared__ dcplx V[kPcaMaxJ][kPcaMaxJ + 1];
  __shared__ int pp[kPcaMaxJ / 2], qq[kPcaMaxJ / 2];
  __shared__ double rc[kPcaMaxJ / 2], rs[kPcaMaxJ / 2];
  __shared__ dcplx re[kPcaMaxJ / 2];   // e^{-i phi}
  __shared__ double red[256];
  __shared__ int order[kPcaMaxJ];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int M = (J + 1) & ~1;          // even number of slots (slot J is a dummy when J is odd)
  for (int i = tid; i < J * J; i += nt) {
    const int r = i / J, c = i % J;
    A[r][c] = dcplx{Cin[i * 2], Cin[i * 2 + 1]};
    V[r][c] = dcplx{r == c ? 1.0 : 0.0, 0.0};
  }
  __syncthreads();
  // Frobenius norm for the stopping rule
  double fro = 0.0;
  for (int i = tid; i < J * J; i += nt) {
    const dcplx v = A[i / J][i % J];
    fro += v.x * v.x + v.y * v.y;
  }
  red[tid] = fro;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  const double tol = 1e-30 * red[0];   // off(A)^2 < 1e-30 ||A||_F^2
  __syncthreads();
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    double off = 0.0;
    for (int i = tid; i < J * J; i += nt) {
      const int r = i / J, c = i % J;
      if (r != c) off += A[r][c].x * A[r][c].x + A[r][c].y * A[r][c].y;
    }
    red[tid] = off;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (tid < o) red[tid] += red[tid + o];
      __syncthreads();
    }
    const bool done = red[0] <= tol;
    __syncthreads();
    if (done) break;
    for (int step = 0; step < M - 1; ++step) {
      // round-robin: slot 0 fixed, slots 1..M-1 rotate
      if (tid < M / 2) {
        auto slot = [&](int k) { return k == 0 ? 0 : 1 + (k - 1 + step) % (M - 1); };
        int p = slot(tid), q = slot(M - 1 - tid);
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        pp[tid] = p;
        qq[tid] = q;
        double c = 1.0, s = 0.0;
        dcplx e{1.0, 0.0};
        if (q < J) {
          const dcplx b = A[p][q];
          const double bm = sqrt(b.x * b.x + b.y * b.y);
          if (bm > 0.0) {
            const double tau = (A[q][q].x - A[p][p].x) / (2.0 * bm);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            e = dcplx{b.x / bm, -b.y / bm};   // e^{-i phi}
          }
        }
        rc[tid] = c;
        rs[tid] = s;
        re[tid] = e;
      }
      __syncthreads();
      // columns: A <- A G, V <- V G (G[p][p] = c, G[p][q] = s, G[q][p] = -s e, G[q][q] = c e)
      for (int i = tid; i < (M / 2) * J; i += nt) {
        const int k = i / J, r = i % J;
        const int p = pp[k], q = qq[k];
        if (q >= J) continue;
        const double c = rc[k], s = rs[k];
        const dcplx e = re[k];
        const dcplx ap = A[r][p], aq = A[r][q];
        const dcplx aqe{aq.x * e.x - aq.y * e.y, aq.x * e.y + aq.y * e.x};
        A[r][p] = dcplx{c * ap.x - s * aqe.x, c * ap.y - s * aqe.y};
        A[r][q] = dcplx{s * ap.x + c * aqe.x, s * ap.y + c * aqe.y};
        const dcplx vp = V[r][p], vq = V[r][q];
        const dcplx vqe{vq.x * e.x - vq.y * e.y, vq.x * e.y + vq.y * e.x};
        V[r][p] = dcplx{c * vp.x - s * vqe.x, c * vp.y - s * vqe.y};
        V[r][q] = dcplx{s * vp.x + c * vqe.x, s * vp.y + c * vqe.y};
      }
      __syncthreads();
      // rows: A <- G^H A (row p: c A_p - s conj(e) A_q; row q: s A_p + c conj(e) A_q)
      for (int i = tid; i < (M / 2) * J; i += nt) {
        const int k = i / J, cidx = i % J;
        const int p = pp[k], q = qq[k];
        if (q >= J) continue;
        const double c = rc[k], s = rs[k];
        const dcplx e = re[k];
        const dcplx ap = A[p][cidx], aq = A[q][cidx];
        const dcplx aqe{aq.x * e.x + aq.y * e.y, aq.y * e.x - aq.x * e.y};   // conj(e) aq
        A[p][cidx] = dcplx{c * ap.x - s * aqe.x, c * ap.y - s * aqe.y};
        A[q][cidx] = dcplx{s * ap.x + c * aqe.x, s * ap.y + c * aqe.y};
      }
      __syncthreads();
    }
  }
  // descending order of the eigenvalues (ties: lower index first)
  for (int i = tid; i < J; i += nt) {
    const double wi = A[i][i].x;
    int rank = 0;
    for (int k = 0; k < J; ++k) {
      const double wk = A[k][k].x;
      if (wk > wi || (wk == wi && k < i)) ++rank;
    }
    order[rank] = i;
  }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0, top = 0.0;
    for (int r = 0; r < J; ++r) {
      const double w = A[order[r]][order[r]].x;
      eig_out[r] = w;
      tot += (w > 0.0 ? w : 0.0);
      if (r < Jc) top += (w > 0.0 ? w : 0.0);
    }
    *energy_out = tot > 0.0 ? top / tot : 1.0;
    *sweeps_out = sweep;
  }
  // top-Jc eigenvectors with the sign convention (largest |v_j|, first index on ties, real-positive)
  for (int k = tid; k < Jc; k += nt) {
    const int col = order[k];
    int m = 0;
    double best = -1.0;
    for (int j = 0; j < J; ++j) {
      const double mag = V[j][col].x * V[j][col].x + V[j][col].y * V[j][col].y;
      if (mag > best) {
        best = mag;
        m = j;
      }
    }
    const double am = sqrt(best);
    const dcplx ph = am > 0.0 ? dcplx{V[m][col].x / am, -V[m][col].y / am} : dcplx{1.0, 0.0};   // conj(v_m)/|v_m|
    for (int j = 0; j < J; ++j) {
      const dcplx v = V[j][col];
      Vout[j * Jc + k] = make_float2((float)(v.x * ph.x - v.y * ph.y), (float)(v.x * ph.y + v.y * ph.x));
    }
  }
}

// ---------------------------------------------------------------- projection
// out[k][n] = sum_j conj(V[j][k]) Y[j][n], channels in ascending order. Each thread owns two
// adjacent samples (one 16-byte load per channel row: coalesced) and a chunk of up to 16 outputs;
// V sits in shared memory, read as float4 = two components (broadcast within a warp), so every
// shared load feeds 4 complex FMAs.
template <int KC>   // outputs per pass (V zero-padded to a multiple of KC: branch-free inner loop)
__global__ void __launch_bounds__(256) pca_apply_kernel(const float2* __restrict__ V, const float2* __restrict__ Y, int J,
                                                        int Jc, long long nsamp, float2* __restrict__ out) {
  __shared__ __align__(16) float2 Vs[kPcaMaxJ * (kPcaMaxJ + 16)];
  const int Jp = ((Jc + KC - 1) / KC) * KC;
  for (int i = threadIdx.x; i < J * Jp; i += blockDim.x) {
    const int j = i / Jp, k = i % Jp;
    Vs[i] = (k < Jc) ? V[j * Jc + k] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const long long npair = (nsamp + 1) / 2;
  const bool vec = (nsamp % 2) == 0;   // 16-byte aligned rows
  for (long long pidx = blockIdx.x * (long long)blockDim.x + threadIdx.x; pidx < npair;
       pidx += (long long)gridDim.x * blockDim.x) {
    const long long n = 2 * pidx;
    const bool two = (n + 1) < nsamp;
    for (int k0 = 0; k0 < Jc; k0 += KC) {
      float2 a0[KC], a1[KC];
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) a0[kk] = a1[kk] = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int j = 0; j < J; ++j) {   // unrolled so four channel loads are in flight together
        float2 y0, y1;
        if (vec) {
          const float4 yy = __ldg(reinterpret_cast<const float4*>(Y + (size_t)j * nsamp + n));
          y0 = make_float2(yy.x, yy.y);
          y1 = make_float2(yy.z, yy.w);
        } else {
          y0 = Y[(size_t)j * nsamp + n];
          y1 = two ? Y[(size_t)j * nsamp + n + 1] : make_float2(0.f, 0.f);
        }
        const float4* vr = reinterpret_cast<const float4*>(Vs + j * Jp + k0);
#pragma unroll
        for (int kp = 0; kp < KC / 2; ++kp) {
          const float4 v = vr[kp];   // components k0+2kp (x, y) and k0+2kp+1 (z, w); conj(v) y
          a0[2 * kp].x = fmaf(v.x, y0.x, fmaf(v.y, y0.y, a0[2 * kp].x));
          a0[2 * kp].y = fmaf(v.x, y0.y, fmaf(-v.y, y0.x, a0[2 * kp].y));
          a1[2 * kp].x = fmaf(v.x, y1.x, fmaf(v.y, y1.y, a1[2 * kp].x));
          a1[2 * kp].y = fmaf(v.x, y1.y, fmaf(-v.y, y1.x, a1[2 * kp].y));
          a0[2 * kp + 1].x = fmaf(v.z, y0.x, fmaf(v.w, y0.y, a0[2 * kp + 1].x));
          a0[2 * kp + 1].y = fmaf(v.z, y0.y, fmaf(-v.w, y0.x, a0[2 * kp + 1].y));
          a1[2 * kp + 1].x = fmaf(v.z, y1.x, fmaf(v.w, y1.y, a1[2 * kp + 1].x));
          a1[2 * kp + 1].y = fmaf(v.z, y1.y, fmaf(-v.w, y1.x, a1[2 * kp + 1].y));
        }
      }
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        if (k0 + kk < Jc) {
          float2* o = out + (size_t)(k0 + kk) * nsamp + n;
          if (vec) {
            *reinterpret_cast<float4*>(o) = make_float4(a0[kk].x, a0[kk].y, a1[kk].x, a1[kk].y);
          } else {
            o[0] = a0[kk];
            if (two) o[1] = a1[kk];
          }
        }
      }
    }
  }
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace
}  // namespace nlv

struct nlinv_pca_s {
  int J = 0, Jc = 0;
  double* part = nullptr;    // [kCovMaxBlocks][4x4 blocks of the upper triangle][16][2]
  double* C = nullptr;       // [J][J][2]
  float2* V = nullptr;       // [J][Jc]
  double* eig = nullptr;     // [J]
  double* energy = nullptr;  // [1]
  int* sweeps = nullptr;
  bool fitted = false;
  std::string err;
  long long launches = 0;
};

using nlv::set_lib_error;

static nlinv_status pfail(nlinv_pca h, nlinv_status s, const std::string& m) {
  if (h) h->err = m;
  set_lib_error(m);
  return s;
}
#define PCU(call)                                                                             \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return pfail(h, NLINV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" nlinv_status nlinv_pca_create(int J, int Jc, nlinv_pca* out) {
  nlinv_pca h = nullptr;
  if (!out) return pfail(h, NLINV_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (J < 1 || J > nlv::kPcaMaxJ) return pfail(h, NLINV_ERR_SIZE, "PCA needs 1 <= J <= 32 channels");
  if (Jc < 1 || Jc > J) return pfail(h, NLINV_ERR_ARG, "PCA needs 1 <= J' <= J (S:530)");
  h = new nlinv_pca_s();
  h->J = J;
  h->Jc = Jc;
  const size_t ntri = (size_t)((J + 3) / 4) * ((J + 3) / 4 + 1) / 2;
  cudaError_t e = cudaMalloc((void**)&h->part, sizeof(double) * 32 * ntri * nlv::kCovMaxBlocks);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->C, sizeof(double) * 2 * J * J);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->V, sizeof(float2) * J * Jc);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->eig, sizeof(double) * (J + 1));
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->energy, sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->sweeps, sizeof(int));
  if (e != cudaSuccess) {
    nlinv_pca_destroy(h);
    return pfail(nullptr, NLINV_ERR_NOMEM, std::string("PCA workspace: ") + cudaGetErrorString(e));
  }
  *out = h;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_pca_destroy(nlinv_pca h) {
  if (!h) return NLINV_OK;
  cudaFree(h->part);
  cudaFree(h->C);
  cudaFree(h->V);
  cudaFree(h->eig);
  cudaFree(h->energy);
  cudaFree(h->sweeps);
  delete h;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_pca_fit(nlinv_pca h, const nlinv_c32* Y, long long nsamp, void* stream) {
  if (!h || !Y) return pfail(h, NLINV_ERR_ARG, "NULL argument to nlinv_pca_fit");
  if (nsamp < 1) return pfail(h, NLINV_ERR_ARG, "nsamp must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  const long long ntile = (nsamp + nlv::kCovTN - 1) / nlv::kCovTN;
  int nblk = nlv::sm_count();
  if (nblk > nlv::kCovMaxBlocks) nblk = nlv::kCovMaxBlocks;
  if ((long long)nblk > ntile) nblk = (int)ntile;
  const float2* y = reinterpret_cast<const float2*>(Y);
  nlv::cov_partial_kernel<<<nblk, nlv::kCovThreads, 0, s>>>(y, h->J, nsamp, h->part);
  PCU(cudaGetLastError());
  const int ntri = ((h->J + 3) / 4) * ((h->J + 3) / 4 + 1) / 2;
  nlv::cov_finish_kernel<<<(ntri * 16 + 255) / 256, 256, 0, s>>>(h->part, nblk, h->J, h->C);
  PCU(cudaGetLastError());
  nlv::jacobi_kernel<<<1, 256, 0, s>>>(h->C, h->J, h->Jc, h->V, h->eig, h->energy, h->sweeps);
  PCU(cudaGetLastError());
  h->launches += 3;
  h->fitted = true;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_pca_result(nlinv_pca h, nlinv_c32* V_host, double* eig_host, double* energy,
                                         double* cov_host) {
  if (!h) return pfail(h, NLINV_ERR_ARG, "NULL handle");
  if (!h->fitted) return pfail(h, NLINV_ERR_STATE, "nlinv_pca_result before nlinv_pca_fit / set_matrix");
  PCU(cudaDeviceSynchronize());
  if (V_host) PCU(cudaMemcpy(V_host, h->V, sizeof(float2) * h->J * h->Jc, cudaMemcpyDeviceToHost));
  if (eig_host) PCU(cudaMemcpy(eig_host, h->eig, sizeof(double) * h->J, cudaMemcpyDeviceToHost));
  if (energy) PCU(cudaMemcpy(energy, h->energy, sizeof(double), cudaMemcpyDeviceToHost));
  if (cov_host) PCU(cudaMemcpy(cov_host, h->C, sizeof(double) * 2 * h->J * h->J, cudaMemcpyDeviceToHost));
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_pca_set_matrix(nlinv_pca h, const nlinv_c32* V_host) {
  if (!h || !V_host) return pfail(h, NLINV_ERR_ARG, "NULL argument to nlinv_pca_set_matrix");
  PCU(cudaMemcpy(h->V, V_host, sizeof(float2) * h->J * h->Jc, cudaMemcpyHostToDevice));
  h->fitted = true;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_pca_apply(nlinv_pca h, const nlinv_c32* Y, long long nsamp, nlinv_c32* out,
                                        void* stream) {
  if (!h || !Y || !out) return pfail(h, NLINV_ERR_ARG, "NULL argument to nlinv_pca_apply");
  if (!h->fitted) return pfail(h, NLINV_ERR_STATE, "nlinv_pca_apply before nlinv_pca_fit / set_matrix");
  if (nsamp < 1) return pfail(h, NLINV_ERR_ARG, "nsamp must be >= 1");
  if ((const void*)Y == (const void*)out) return pfail(h, NLINV_ERR_ARG, "in-place apply is not supported");
  cudaStream_t s = (cudaStream_t)stream;
  long long nb = ((nsamp + 1) / 2 + 255) / 256;
  const long long cap = 8LL * nlv::sm_count();
  if (nb > cap) nb = cap;
  const float2* y = reinterpret_cast<const float2*>(Y);
  float2* o = reinterpret_cast<float2*>(out);
  if (h->Jc <= 4) nlv::pca_apply_kernel<4><<<(int)nb, 256, 0, s>>>(h->V, y, h->J, h->Jc, nsamp, o);
  else if (h->Jc <= 8) nlv::pca_apply_kernel<8><<<(int)nb, 256, 0, s>>>(h->V, y, h->J, h->Jc, nsamp, o);
  else if (h->Jc <= 12) nlv::pca_apply_kernel<12><<<(int)nb, 256, 0, s>>>(h->V, y, h->J, h->Jc, nsamp, o);
  else nlv::pca_apply_kernel<16><<<(int)nb, 256, 0, s>>>(h->V, y, h->J, h->Jc, nsamp, o);
  PCU(cudaGetLastError());
  h->launches += 1;
  return NLINV_OK;
}

extern "C" const char* nlinv_pca_last_error(nlinv_pca h) { return h ? h->err.c_str() : ""; }
extern "C" long long nlinv_pca_launch_count(nlinv_pca h) { return h ? h->launches : 0; }
