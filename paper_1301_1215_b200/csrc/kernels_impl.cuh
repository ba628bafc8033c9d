// sm_100a kernels of the NLINV / IRGNM hot path (§3.1-3.2).
//
// Per coil j the normal operator N(p) = DF^H DF p + alpha p (Eq. 3) is five fused
// passes over the doubled grid, each a batch of 1D FFTs with its pointwise work
// fused into prologue/epilogue ("point-wise matrix operations"):
//   K1 col : t = w^-1 p_chat            -> column IFFT -> keep Omega rows
//   K2 row : row IFFT -> dc; z = M(p_rho c + rho dc) -> row FFT
//   K3 col : column FFT -> x P_k -> column IFFT -> keep Omega rows   (the PSF convolution)
//   K4 row : row IFFT -> u; S += conj(c) u (sum over coils, Table 1 "sum c_j"); v = conj(rho) u -> row FFT
//   K5 col : column FFT -> Ap_chat = w^-1 . + alpha p_chat; <p, Ap> partial
// Only the n Omega rows/columns of the image-side arrays are ever stored (M_Omega follows
// every image-side step), which halves every row pass and every column-pass input.
//
// Centred unitary DFT (R1): per dimension F_c = (-1)^k FFT((-1)^i .) / sqrt(L) for
// L % 4 == 0; each 2D transform carries 1/L once.
#pragma once
#include "fft.cuh"
#include "nlinv_kernels.cuh"

namespace nlv {

// ------------------------------------------------------------------ launch geometry
template <int L>
struct ColGeo {
  static constexpr int T = Cfg<L>::T;
  static constexpr int c0 = (256 / T) < 32 ? (256 / T) : 32;
  static constexpr int CW = (L % c0 == 0) ? c0 : ((L % 16 == 0 && c0 >= 16) ? 16 : 8);
  static constexpr int THREADS = CW * T;
  static constexpr size_t SMEM = sizeof(float2) * (size_t)L * (CW + 1) + 64 * sizeof(double);
};

template <int L>
struct RowGeo {
  static constexpr int T = Cfg<L>::T;
  static constexpr int GCMAX = (L >= 512) ? 8 : 16;  // coil groups per CTA
  static size_t smem(int gc) { return sizeof(float2) * (size_t)L * (gc + 1) + sizeof(float2) * (L / 2) + 64 * sizeof(double); }
};

struct SyncBlock {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct SyncWarp {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

template <int CW>
struct ColBuf {
  float2* s;
  int c;
  __device__ __forceinline__ float2& operator()(int i) const { return s[i * CW + c]; }
};
struct RowBuf {
  float2* s;
  __device__ __forceinline__ float2& operator()(int i) const { return s[i]; }
};

__device__ __forceinline__ float sgn_of(int i) { return (i & 1) ? -1.0f : 1.0f; }

// Omega membership of register e (compile-time after unrolling; L/R divides L/4 for R % 4 == 0)
template <int L>
__device__ __forceinline__ constexpr bool in_is_omega(int e) {
  constexpr int R = Cfg<L>::R0;
  return (e % R) * (L / R) >= L / 4 && (e % R) * (L / R) < 3 * L / 4;
}
template <int L>
__device__ __forceinline__ constexpr bool out_is_omega(int e) {
  constexpr int R = Sched<L>::RL;
  return (e % R) * (L / R) >= L / 4 && (e % R) * (L / R) < 3 * L / 4;
}

// ------------------------------------------------------------------ deterministic reductions
// Block sum in a fixed tree (warp xor-shuffles, then warps in index order). Result valid in
// thread 0. red must hold 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
  }
  return s;
}

// Grid-level deterministic finish: every CTA publishes NV partials; the last CTA to arrive
// sums them in block-index order and writes out[k] = sum. The counter is re-armed for replay.
template <int NV>
__device__ __forceinline__ void grid_finish(const double (&v)[NV], double* partials, unsigned* counter,
                                            double* scal_w, const int (&slot)[NV], double* red) {
  const unsigned nblk = gridDim.x * gridDim.y;
  const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
  __shared__ bool is_last;
  double s[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) s[k] = block_sum(v[k], red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * kMaxRedBlocks + bid] = s[k];
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    is_last = (ticket == nblk - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (threadIdx.x < 32) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double acc = 0.0;
        const volatile double* pv = partials + k * kMaxRedBlocks;
        for (unsigned i = threadIdx.x; i < nblk; i += 32) acc += pv[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0 && slot[k] >= 0) scal_w[slot[k]] = acc;
      }
      if (threadIdx.x == 0) *counter = 0u;
    }
  }
}

__device__ __forceinline__ float cg_beta(const double* scal, int i) {
  if (i <= 0) return 0.0f;
  const double rr = scal[SC_RR_RHO + i] + scal[SC_RR_CHAT + i];
  const double rp = scal[SC_RR_RHO + i - 1] + scal[SC_RR_CHAT + i - 1];
  return rp != 0.0 ? (float)(rr / rp) : 0.0f;
}
__device__ __forceinline__ float cg_gamma(const double* scal, int i) {
  const double rr = scal[SC_RR_RHO + i] + scal[SC_RR_CHAT + i];
  const double pap = scal[SC_PAP_RHO + i] + scal[SC_PAP_CHAT + i];
  return rr != 0.0 ? (float)(rr / pap) : 0.0f;
}

// ------------------------------------------------------------------ column kernels
template <int L, int MODE>
__global__ void __launch_bounds__(ColGeo<L>::THREADS) col_kernel(ColArgs a, const float2* __restrict__ twg) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E, CW = ColGeo<L>::CW, NT = ColGeo<L>::THREADS;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t N = (size_t)L * L, H = (size_t)n * L;
  constexpr float invL = 1.0f / (float)L;
  constexpr int DIR_FIRST = (MODE == CK_IFFT_W || MODE == CK_IFFT_W_CG || MODE == CK_ADJ1) ? +1 : -1;

  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  double* red = reinterpret_cast<double*>(xb + (size_t)L * CW);

  const int tid = threadIdx.x, c = tid % CW, t = tid / CW;
  const int x = blockIdx.x * CW + c;
  const int j = blockIdx.y;

  if constexpr (MODE == CK_IFFT_W_CG) {
    if (j == a.J) {  // rho-block slice of the fused CG direction update p = r + beta p
      const float beta = cg_beta(a.scal, a.iter);
      for (int y = t; y < L; y += T) {
        const size_t i = (size_t)y * L + x;
        const float2 rv = a.rho_r[i], pv = a.rho_p[i];
        a.rho_p[i] = make_float2(fmaf(beta, pv.x, rv.x), fmaf(beta, pv.y, rv.y));
      }
      return;
    }
  }
  for (int i = tid; i < L; i += NT) tw[i] = twg[i];
  __syncthreads();

  ColBuf<CW> buf{xb, c};
  float2 v[E];
  double acc = 0.0;

  // ---------------- prologue: pass-0 input pattern, index = row
  if constexpr (MODE == CK_IFFT_W || MODE == CK_IFFT_W_CG) {
    const float beta = (MODE == CK_IFFT_W_CG) ? cg_beta(a.scal, a.iter) : 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int yr = S::in_idx(t, e);
      const size_t i = (size_t)yr * L + x;
      float2 s;
      if constexpr (MODE == CK_IFFT_W_CG) {
        const float2 rv = a.r[j * N + i], pv = a.p[j * N + i];
        s = make_float2(fmaf(beta, pv.x, rv.x), fmaf(beta, pv.y, rv.y));
        a.p[j * N + i] = s;
      } else {
        s = a.src[j * N + i];
      }
      v[e] = cscale(s, a.winv[i] * sgn_of(yr));
    }
  } else if constexpr (MODE == CK_ADJ1) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int yr = S::in_idx(t, e);
      const size_t i = (size_t)yr * L + x;
      const float2 s = a.in[j * N + i];
      v[e] = a.mask[i] ? cneg_if(s, yr & 1) : make_float2(0.f, 0.f);
    }
  } else {  // half-image input: only Omega rows are non-zero
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (in_is_omega<L>(e)) {
        const int yr = S::in_idx(t, e);
        v[e] = cneg_if(a.in[j * H + (size_t)(yr - q) * L + x], yr & 1);
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
  }

  fft<L, DIR_FIRST>(v, t, tw, buf, SyncBlock{});

  // ---------------- middle: k-space pointwise (registers hold output pattern, index = k)
  if constexpr (MODE == CK_PSF || MODE == CK_RESADJ) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      const size_t i = (size_t)k * L + x;
      if constexpr (MODE == CK_PSF) {
        // (-1)^k post-sign of the FFT and pre-sign of the IFFT cancel
        v[e] = a.mask[i] ? v[e] : make_float2(0.f, 0.f);
      } else {
        // r = P (y - F x), F x = (-1)^k G; the IFFT consumes (-1)^k r = P((-1)^k y - G)
        float2 rr = make_float2(0.f, 0.f);
        if (a.mask[i]) {
          const float2 yv = cneg_if(a.y[j * N + i], k & 1);
          rr = csub(yv, v[e]);
          acc += (double)rr.x * rr.x + (double)rr.y * rr.y;
        }
        v[e] = rr;
      }
    }
    out_to_in<L>(v, t, buf, SyncBlock{});
    fft<L, +1>(v, t, tw, buf, SyncBlock{});
  }

  // ---------------- epilogue: last-pass output pattern, index = row k
  if constexpr (MODE == CK_IFFT_W || MODE == CK_IFFT_W_CG || MODE == CK_PSF || MODE == CK_RESADJ ||
                MODE == CK_ADJ1) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        a.out[j * H + (size_t)(k - q) * L + x] = cscale(v[e], invL * sgn_of(k));
      }
    }
  } else if constexpr (MODE == CK_FWDP) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      const size_t i = (size_t)k * L + x;
      a.out[j * N + i] = a.mask[i] ? cneg_if(v[e], k & 1) : make_float2(0.f, 0.f);
    }
  } else {  // CK_FFT_W_*
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      const size_t i = (size_t)k * L + x;
      const float2 val = cscale(v[e], a.winv[i] * sgn_of(k));
      if constexpr (MODE == CK_FFT_W_NORMAL) {
        const float2 pv = a.src2[j * N + i];
        const float2 o = make_float2(fmaf(a.alpha, pv.x, val.x), fmaf(a.alpha, pv.y, val.y));
        a.out[j * N + i] = o;
        acc += (double)pv.x * o.x + (double)pv.y * o.y;
      } else if constexpr (MODE == CK_FFT_W_RHS) {
        const float2 xc = a.src[j * N + i], xr = a.src2[j * N + i];
        const float2 d = csub(xc, xr);
        const float2 b = make_float2(fmaf(-a.alpha, d.x, val.x), fmaf(-a.alpha, d.y, val.y));
        a.r[j * N + i] = b;
        a.p[j * N + i] = b;
        acc += (double)b.x * b.x + (double)b.y * b.y;
      } else {
        a.out[j * N + i] = val;
      }
    }
  }

  if constexpr (MODE == CK_RESADJ || MODE == CK_FFT_W_NORMAL || MODE == CK_FFT_W_RHS) {
    if (a.partials != nullptr) {
      const double vv[1] = {acc};
      const int sl[1] = {a.out_slot};
      grid_finish<1>(vv, a.partials, a.counter, a.scal_w, sl, red);
    }
  }
}

// ------------------------------------------------------------------ row kernels
template <int L, int MODE>
__global__ void __launch_bounds__(512) row_kernel(RowArgs a, const float2* __restrict__ twg) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t H = (size_t)n * L, Q = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;

  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xbase = tw + L;                                  // [gc][L]
  float2* accs = xbase + (size_t)L * a.gc;                 // [n] coil-sum accumulator

  const int yy = blockIdx.x, row = q + yy;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int g = tid / T, t = tid % T;
  RowBuf buf{xbase + (size_t)g * L};

  for (int i = tid; i < L; i += nt) tw[i] = twg[i];
  if constexpr (MODE == RK_K4 || MODE == RK_RSS)
    for (int i = tid; i < n; i += nt) accs[i] = make_float2(0.f, 0.f);
  if constexpr (MODE == RK_SETPOINT || MODE == RK_SETPOINT_FWD || MODE == RK_RSS)
    for (int i = tid; i < n; i += nt) a.rho_omega[yy * n + i] = a.xrho[(size_t)row * L + q + i];
  __syncthreads();

  for (int j0 = 0; j0 < a.J; j0 += a.gc) {
    const int j = j0 + g;
    const bool active = j < a.J;
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int xi = S::in_idx(t, e);
      v[e] = make_float2(0.f, 0.f);
      if (active) v[e] = cneg_if(a.in[j * H + (size_t)yy * L + xi], xi & 1);
    }
    fft<L, +1>(v, t, tw, buf, SyncWarp{});
    // v[e] now holds (-1)^k x (row IFFT), k = S::out_idx(t, e); only Omega columns are kept

    if constexpr (MODE == RK_SETPOINT || MODE == RK_SETPOINT_FWD || MODE == RK_RSS) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        if (out_is_omega<L>(e)) {
          const float2 cv = cneg_if(v[e], k & 1);
          if (active) a.c_omega[j * Q + (size_t)yy * n + (k - q)] = cv;
          if constexpr (MODE == RK_SETPOINT_FWD) {
            const float2 rv = a.xrho[(size_t)row * L + k];
            v[e] = cscale(cmul(rv, cv), invL * sgn_of(k));
          } else if constexpr (MODE == RK_RSS) {
            buf(k - q) = make_float2(cv.x * cv.x + cv.y * cv.y, 0.f);
          }
        } else {
          v[e] = make_float2(0.f, 0.f);
        }
      }
    } else if constexpr (MODE == RK_K2) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        if (out_is_omega<L>(e) && active) {
          const float2 dc = cneg_if(v[e], k & 1);
          const float2 cv = a.c_omega[j * Q + (size_t)yy * n + (k - q)];
          const float2 rv = a.rho_omega[(size_t)yy * n + (k - q)];
          const float2 pr = a.prho[(size_t)row * L + k];
          const float2 z = cadd(cmul(pr, cv), cmul(rv, dc));
          v[e] = cscale(z, invL * sgn_of(k));
        } else {
          v[e] = make_float2(0.f, 0.f);
        }
      }
    } else if constexpr (MODE == RK_K4) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        if (out_is_omega<L>(e)) {
          const float2 u = cneg_if(v[e], k & 1);
          float2 term = make_float2(0.f, 0.f);
          if (active) {
            const float2 cv = a.c_omega[j * Q + (size_t)yy * n + (k - q)];
            term = cmulc(cv, u);
          }
          buf(k - q) = term;
          const float2 rv = a.rho_omega[(size_t)yy * n + (k - q)];
          v[e] = cscale(cmulc(rv, u), invL * sgn_of(k));
        } else {
          v[e] = make_float2(0.f, 0.f);
        }
      }
    }

    if constexpr (MODE == RK_K4 || MODE == RK_RSS) {
      // ordered sum over the coils of this chunk (ascending coil index)
      __syncthreads();
      for (int xx = tid; xx < n; xx += nt) {
        float2 s = accs[xx];
        for (int gg = 0; gg < a.gc && j0 + gg < a.J; ++gg) s = cadd(s, xbase[(size_t)gg * L + xx]);
        accs[xx] = s;
      }
      __syncthreads();
    }

    if constexpr (MODE == RK_SETPOINT_FWD || MODE == RK_K2 || MODE == RK_K4) {
      out_to_in<L>(v, t, buf, SyncWarp{});
      fft<L, -1>(v, t, tw, buf, SyncWarp{});
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int k = S::out_idx(t, e);
          a.out[j * H + (size_t)yy * L + k] = cneg_if(v[e], k & 1);
        }
      }
    }
  }

  if constexpr (MODE == RK_K4) {
    __syncthreads();
    for (int i = tid; i < n; i += nt) a.S[(size_t)yy * n + i] = accs[i];
  } else if constexpr (MODE == RK_RSS) {
    __syncthreads();
    for (int i = tid; i < n; i += nt) a.rss[(size_t)yy * n + i] = accs[i].x;
  }
}

// ------------------------------------------------------------------ dispatch
template <int L, int MODE>
static cudaError_t launch_col_t(const ColArgs& a, const float2* tw, cudaStream_t s) {
  auto kern = col_kernel<L, MODE>;
  const size_t smem = ColGeo<L>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int gy = (MODE == CK_IFFT_W_CG) ? a.J + 1 : a.J;
  dim3 grid(L / ColGeo<L>::CW, gy);
  kern<<<grid, ColGeo<L>::THREADS, smem, s>>>(a, tw);
  return cudaGetLastError();
}

template <int L>
static cudaError_t launch_col_l(int mode, const ColArgs& a, const float2* tw, cudaStream_t s) {
  switch (mode) {
    case CK_IFFT_W: return launch_col_t<L, CK_IFFT_W>(a, tw, s);
    case CK_IFFT_W_CG: return launch_col_t<L, CK_IFFT_W_CG>(a, tw, s);
    case CK_FWDP: return launch_col_t<L, CK_FWDP>(a, tw, s);
    case CK_PSF: return launch_col_t<L, CK_PSF>(a, tw, s);
    case CK_RESADJ: return launch_col_t<L, CK_RESADJ>(a, tw, s);
    case CK_ADJ1: return launch_col_t<L, CK_ADJ1>(a, tw, s);
    case CK_FFT_W_NORMAL: return launch_col_t<L, CK_FFT_W_NORMAL>(a, tw, s);
    case CK_FFT_W_RHS: return launch_col_t<L, CK_FFT_W_RHS>(a, tw, s);
    case CK_FFT_W_ADJ: return launch_col_t<L, CK_FFT_W_ADJ>(a, tw, s);
  }
  return cudaErrorInvalidValue;
}

template <int L, int MODE>
static cudaError_t launch_row_t(const RowArgs& a0, const float2* tw, cudaStream_t s) {
  RowArgs a = a0;
  constexpr int T = Cfg<L>::T;
  int gc = a.J < RowGeo<L>::GCMAX ? a.J : RowGeo<L>::GCMAX;
  while ((gc * T) % 32 != 0) ++gc;  // whole warps
  a.gc = gc;
  const size_t smem = RowGeo<L>::smem(gc);
  auto kern = row_kernel<L, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<L / 2, gc * T, smem, s>>>(a, tw);
  return cudaGetLastError();
}

template <int L>
static cudaError_t launch_row_l(int mode, const RowArgs& a, const float2* tw, cudaStream_t s) {
  switch (mode) {
    case RK_SETPOINT: return launch_row_t<L, RK_SETPOINT>(a, tw, s);
    case RK_SETPOINT_FWD: return launch_row_t<L, RK_SETPOINT_FWD>(a, tw, s);
    case RK_RSS: return launch_row_t<L, RK_RSS>(a, tw, s);
    case RK_K2: return launch_row_t<L, RK_K2>(a, tw, s);
    case RK_K4: return launch_row_t<L, RK_K4>(a, tw, s);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ plain batched 2D transform
// (debug / micro-benchmark entry: centred unitary F_c or F_c^H of `batch` images)
template <int L, int DIR>
__global__ void __launch_bounds__(256) fft_rows_tw_kernel(const float2* __restrict__ in, float2* out, int nrows,
                                                         const float2* __restrict__ twg) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E;
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
  __syncthreads();
  const int gpc = blockDim.x / T;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const long long rowi = (long long)blockIdx.x * gpc + g;
  RowBuf buf{xb + (size_t)g * L};
  float2 v[E];
  const bool active = rowi < nrows;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int xi = S::in_idx(t, e);
    v[e] = active ? cneg_if(in[rowi * L + xi], xi & 1) : make_float2(0.f, 0.f);
  }
  fft<L, DIR>(v, t, tw, buf, SyncWarp{});
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      out[rowi * L + k] = cneg_if(v[e], k & 1);
    }
  }
}

template <int L, int DIR>
__global__ void __launch_bounds__(ColGeo<L>::THREADS) fft_cols_tw_kernel(float2* data, const float2* __restrict__ twg) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E, CW = ColGeo<L>::CW;
  constexpr size_t N = (size_t)L * L;
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
  __syncthreads();
  const int tid = threadIdx.x, c = tid % CW, t = tid / CW;
  const int x = blockIdx.x * CW + c;
  float2* d = data + (size_t)blockIdx.y * N;
  ColBuf<CW> buf{xb, c};
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int yr = S::in_idx(t, e);
    v[e] = cneg_if(d[(size_t)yr * L + x], yr & 1);
  }
  fft<L, DIR>(v, t, tw, buf, SyncBlock{});
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = S::out_idx(t, e);
    d[(size_t)k * L + x] = cscale(v[e], (1.0f / (float)L) * sgn_of(k));
  }
}

template <int L>
static cudaError_t launch_fft2d_l(const float2* in, float2* out, int batch, int inverse, const float2* tw,
                                  cudaStream_t s) {
  constexpr int T = Cfg<L>::T;
  const int gpc = 256 / T;
  const int nrows = batch * L;
  const size_t rsm = sizeof(float2) * (size_t)L * (gpc + 1);
  const size_t csm = ColGeo<L>::SMEM;
  cudaError_t e;
  if (inverse) {
    auto rk = fft_rows_tw_kernel<L, +1>;
    auto ck = fft_cols_tw_kernel<L, +1>;
    if ((e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm)) != cudaSuccess) return e;
    rk<<<(nrows + gpc - 1) / gpc, gpc * T, rsm, s>>>(in, out, nrows, tw);
    ck<<<dim3(L / ColGeo<L>::CW, batch), ColGeo<L>::THREADS, csm, s>>>(out, tw);
  } else {
    auto rk = fft_rows_tw_kernel<L, -1>;
    auto ck = fft_cols_tw_kernel<L, -1>;
    if ((e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm)) != cudaSuccess) return e;
    rk<<<(nrows + gpc - 1) / gpc, gpc * T, rsm, s>>>(in, out, nrows, tw);
    ck<<<dim3(L / ColGeo<L>::CW, batch), ColGeo<L>::THREADS, csm, s>>>(out, tw);
  }
  return cudaGetLastError();
}

// Per-grid-size entry points, defined in one translation unit per size (inst.cu -DNLV_L=...).
#define NLV_DECLARE(L)                                                                           \
  cudaError_t launch_col_##L(int mode, const ColArgs& a, const float2* tw, cudaStream_t s);     \
  cudaError_t launch_row_##L(int mode, const RowArgs& a, const float2* tw, cudaStream_t s);     \
  cudaError_t launch_fft2d_##L(const float2* in, float2* out, int batch, int inverse, const float2* tw, \
                               cudaStream_t s);                                                 \
  int col_tiles_##L();
#define NLV_INSTANTIATE(L)                                                                       \
  cudaError_t launch_col_##L(int mode, const ColArgs& a, const float2* tw, cudaStream_t s) {    \
    return launch_col_l<L>(mode, a, tw, s);                                                      \
  }                                                                                              \
  cudaError_t launch_row_##L(int mode, const RowArgs& a, const float2* tw, cudaStream_t s) {    \
    return launch_row_l<L>(mode, a, tw, s);                                                      \
  }                                                                                              \
  cudaError_t launch_fft2d_##L(const float2* in, float2* out, int batch, int inverse, const float2* tw, \
                               cudaStream_t s) {                                                 \
    return launch_fft2d_l<L>(in, out, batch, inverse, tw, s);                                    \
  }                                                                                              \
  int col_tiles_##L() { return L / ColGeo<L>::CW; }

#define NLV_FOR_EACH_NG(X) X(16) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384) X(512) X(768) X(1024)
NLV_FOR_EACH_NG(NLV_DECLARE)

}  // namespace nlv
