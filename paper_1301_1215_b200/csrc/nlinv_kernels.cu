// Non-templated kernels (rho block, CG vector update, frame output) and the grid-size
// dispatch of the templated FFT-pass kernels (kernels_impl.cuh, one TU per size in inst.cu).
#include <cstdlib>

#include "kernels_impl.cuh"

namespace nlv {

int k4_chunk_override() {
  static const int v = [] {
    const char* e = std::getenv("NLINV_K4CHUNK");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

int row_pairs_override() {
  static const int v = [] {
    const char* e = std::getenv("NLINV_ROWPAIRS");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

int fft_radices(int ng, int* R) {
#define X(L) if (ng == L) { R[0] = Cfg<L>::R0; R[1] = Cfg<L>::R1; R[2] = Cfg<L>::R2; R[3] = Cfg<L>::R3; return Cfg<L>::NP; }
  NLV_FOR_EACH_NG(X)
#undef X
  return 0;
}

int k4_planes(int ng, int J) {
#define X(L) if (ng == L) { const int c = k4_chunk_t<L>(J); return (J + c - 1) / c; }
  NLV_FOR_EACH_NG(X)
#undef X
  return J;
}

bool k2_one_enabled() {   // NLINV_K2ONE=0: K2 always with the two-CTA register bound
  static const bool on = [] {
    const char* e = std::getenv("NLINV_K2ONE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NLINV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ------------------------------------------------------------------ rho-block kernels
constexpr int kVecThreads = 256;

// Newton update after L CG iterations: x += dx + gamma_{L-1} p_{L-1}
// (dx holds the steps of iterations 0 .. L-2, folded into K1; iter = L).
__global__ void __launch_bounds__(kVecThreads) newton_update_kernel(VecArgs a) {
  pdl_wait();
  pdl_trigger();
  const float gamma = cg_gamma(a.scal, a.iter - 1);
  const bool hasdx = a.iter > 1;
  const long long n2 = a.ntot / 2, stride = (long long)gridDim.x * blockDim.x;
  const float4* p4 = reinterpret_cast<const float4*>(a.p);
  const float4* dx4 = reinterpret_cast<const float4*>(a.dx);
  float4* x4 = reinterpret_cast<float4*>(a.x);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += stride) {
    const float4 pv = p4[i];
    const float4 d = hasdx ? dx4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 xv = x4[i];
    xv.x += fmaf(gamma, pv.x, d.x); xv.y += fmaf(gamma, pv.y, d.y);
    xv.z += fmaf(gamma, pv.z, d.z); xv.w += fmaf(gamma, pv.w, d.w);
    x4[i] = xv;
  }
}

// CG residual update r_{i+1} = r_i - gamma_i A p_i and <r_{i+1}, r_{i+1}> (rho, chat parts)
__global__ void __launch_bounds__(kVecThreads) r_update_kernel(VecArgs a) {
  __shared__ double red[32];
  pdl_wait();
  pdl_trigger();
  const float gamma = cg_gamma(a.scal, a.iter);
  double acc_rho = 0.0, acc_chat = 0.0;
  const long long n2 = a.ntot / 2, stride = (long long)gridDim.x * blockDim.x;
  const float4* ap4 = reinterpret_cast<const float4*>(a.Ap);
  float4* r4 = reinterpret_cast<float4*>(a.r);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += stride) {
    const float4 av = ap4[i];
    float4 rv = r4[i];
    rv.x = fmaf(-gamma, av.x, rv.x); rv.y = fmaf(-gamma, av.y, rv.y);
    rv.z = fmaf(-gamma, av.z, rv.z); rv.w = fmaf(-gamma, av.w, rv.w);
    r4[i] = rv;
    const double sq = (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
    if (2 * i < a.nrho) acc_rho += sq; else acc_chat += sq;
  }
  const double vv[2] = {acc_rho, acc_chat};
  const int sl[2] = {SC_RR_RHO + a.iter + 1, SC_RR_CHAT + a.iter + 1};
  grid_finish<2>(vv, a.partials, a.counter, a.scal_w, sl, red);
}

// frame output: image = crop_Omega(rho) . sqrt(sum_j |c_j|^2), planes summed in order
__global__ void image_kernel(const float2* __restrict__ rho_omega, const float* __restrict__ rss, int nplanes,
                             float2* img, int Q) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < nplanes; ++j) s += rss[(size_t)j * Q + i];
    img[i] = cscale(rho_omega[i], sqrtf(s));
  }
}

// generic two-phase peer exchange (see XPeers): arrive with this rank's scalars in its
// window, wait for every rank, reduce (sums in ascending rank order, or rank 0's value for the
// replicated rho parts), ack, wait for every rank's ack (every window buffer is reusable after it)
__global__ void __launch_bounds__(1024) xchg_kernel(XchgArgs a) {
  __shared__ unsigned long long s_e;
  pdl_wait();
  char* own = a.xp.win[a.xp.rank];
  const int nv = a.nsum + a.nr0;
  double* xs = xw_xs(own);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) xs[i] = a.scal[a.src[i]];
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long e = x_epoch(a.xp, XK_A) + 1;
    x_publish(a.xp, XK_A, e);
    x_wait_all(a.xp, XK_A, e);
    s_e = e;
  }
  __syncthreads();
  double val = 0.0;
  if ((int)threadIdx.x < a.nsum) {
    for (int h = 0; h < a.xp.G; ++h) val += __ldcv(xw_xs(a.xp.win[h]) + threadIdx.x);
  } else if ((int)threadIdx.x < nv) {
    val = __ldcv(xw_xs(a.xp.win[0]) + threadIdx.x);
  }
  if (a.rss_out != nullptr) {
    for (int i = threadIdx.x; i < a.Q; i += blockDim.x) {
      float sacc = 0.f;
      for (int h = 0; h < a.xp.G; ++h) sacc += __ldcv(xw_rss(a.xp.win[h], (size_t)a.Q) + i);
      a.rss_out[i] = sacc;
    }
  }
  if ((int)threadIdx.x < nv) a.scal[a.dst[threadIdx.x]] = val;
  __syncthreads();
  if (threadIdx.x == 0) {
    x_publish(a.xp, XK_B, s_e);
    x_wait_all(a.xp, XK_B, s_e);
  }
}
cudaError_t launch_xchg(const XchgArgs& a, cudaStream_t s) {
  return launch_k(xchg_kernel, dim3(1), dim3(1024), 0, s, a);
}

// micro-benchmark kernel (the paper's axpy of Fig. 4): y = a x + y, float4
// vectorised, grid sized to the SM count (persistent grid-stride loop)
__global__ void __launch_bounds__(256) axpy_kernel(float a, const float4* __restrict__ x, float4* __restrict__ y,
                                                   long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 xv = x[i];
    float4 yv = y[i];
    yv.x = fmaf(a, xv.x, yv.x);
    yv.y = fmaf(a, xv.y, yv.y);
    yv.z = fmaf(a, xv.z, yv.z);
    yv.w = fmaf(a, xv.w, yv.w);
    y[i] = yv;
  }
}
cudaError_t launch_axpy(float a, const float* x, float* y, long long n, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  axpy_kernel<<<nsm * 8, 256, 0, s>>>(a, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n / 4);
  return cudaGetLastError();
}

// local coil sums before the cross-rank all-reduce (world > 1)
__global__ void coil_sum_kernel(const float2* __restrict__ S_all, int J, float2* S, int Q) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += gridDim.x * blockDim.x) {
    float2 s = make_float2(0.f, 0.f);
    for (int j = 0; j < J; ++j) s = cadd(s, S_all[(size_t)j * Q + i]);
    S[i] = s;
  }
}
__global__ void rss_sum_kernel(const float* __restrict__ rss_all, int J, float* rss, int Q) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < J; ++j) s += rss_all[(size_t)j * Q + i];
    rss[i] = s;
  }
}

bool supported_ng(int ng) {
#define X(L) if (ng == L) return true;
  NLV_FOR_EACH_NG(X)
#undef X
  return false;
}

cudaError_t launch_col(int ng, int mode, const ColArgs& a, const float2* tw, cudaStream_t s) {
#define X(L) if (ng == L) return launch_col_##L(mode, a, tw, s);
  NLV_FOR_EACH_NG(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_row(int ng, int mode, const RowArgs& a, const float2* tw, cudaStream_t s) {
#define X(L) if (ng == L) return launch_row_##L(mode, a, tw, s);
  NLV_FOR_EACH_NG(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_fft2d(int ng, const float2* in, float2* out, int batch, int inverse, const float2* tw,
                         float2* /*tmp*/, cudaStream_t s) {
#define X(L) if (ng == L) return launch_fft2d_##L(in, out, batch, inverse, tw, s);
  NLV_FOR_EACH_NG(X)
#undef X
  return cudaErrorInvalidValue;
}

static int vec_grid(long long n) {
  long long b = (n + kVecThreads - 1) / kVecThreads;
  const long long cap = 148 * 4;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_r_update(int /*ng*/, const VecArgs& a, cudaStream_t s) {
  return launch_k(r_update_kernel, dim3(vec_grid(a.ntot / 2)), dim3(kVecThreads), 0, s, a);
}
cudaError_t launch_newton_update(int /*ng*/, const VecArgs& a, cudaStream_t s) {
  return launch_k(newton_update_kernel, dim3(vec_grid(a.ntot / 2)), dim3(kVecThreads), 0, s, a);
}
__global__ void init_x_kernel(float2* x, long long nrho, long long ntot) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ntot; i += (long long)gridDim.x * blockDim.x)
    x[i] = make_float2(i < nrho ? 1.0f : 0.0f, 0.0f);
}
// ------------------------------------------------------------------ P_k -> sorted index list (a0)
// Stream compaction of the sampling mask into ascending linear indices (integer-exact):
// pass 1 counts the sampled cells of each 4096-cell chunk, pass 2 gives every chunk its offset
// (ordered prefix of the counts) and writes its indices in order with warp ballots.
constexpr int kMaskChunk = 4096;
__global__ void __launch_bounds__(256) mask_count_kernel(const uint8_t* __restrict__ mask, int N, int* counts) {
  __shared__ int red[8];
  pdl_wait();
  const int base = blockIdx.x * kMaskChunk;
  int c = 0;
  for (int i = threadIdx.x; i < kMaskChunk; i += 256)
    if (base + i < N && mask[base + i]) ++c;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) mask_scatter_kernel(const uint8_t* __restrict__ mask, int N,
                                                           const int* __restrict__ counts, int* idx, int* nnz) {
  __shared__ int s_off, s_warp[8];
  pdl_wait();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int b = 0; b < (int)blockIdx.x; ++b) o += counts[b];
    s_off = o;
    if (blockIdx.x == gridDim.x - 1) *nnz = o + counts[blockIdx.x];
  }
  __syncthreads();
  const int base = blockIdx.x * kMaskChunk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int off = s_off;
  for (int i0 = 0; i0 < kMaskChunk; i0 += 256) {
    const int i = base + i0 + threadIdx.x;
    const bool m = (i < N) && mask[i];
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (lane == 0) s_warp[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int ww = 0; ww < 8; ++ww) {
      if (ww < w) before += s_warp[ww];
      tot += s_warp[ww];
    }
    if (m) idx[off + before + __popc(bal & ((1u << lane) - 1u))] = i;
    off += tot;
    __syncthreads();
  }
}

cudaError_t launch_mask_compact(const uint8_t* mask, int N, int* counts, int* idx, int* nnz, cudaStream_t s) {
  const int nb = (N + kMaskChunk - 1) / kMaskChunk;
  cudaError_t e = launch_k(mask_count_kernel, dim3(nb), dim3(256), 0, s, mask, N, counts);
  if (e != cudaSuccess) return e;
  return launch_k(mask_scatter_kernel, dim3(nb), dim3(256), 0, s, mask, N, (const int*)counts, idx, nnz);
}
int mask_count_blocks(int N) { return (N + kMaskChunk - 1) / kMaskChunk; }

// compact frame ingest (a1): y_j[idx[s]] = samples_j[s]; cells off P_k are never read
__global__ void scatter_samples_kernel(const float2* __restrict__ samples, const int* __restrict__ idx,
                                       const int* __restrict__ nnz_p, int nnz_cap, int J, size_t N, float2* y) {
  pdl_wait();
  const int nnz = *nnz_p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)J * nnz;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / nnz), s = (int)(i % nnz);
    y[(size_t)j * N + idx[s]] = samples[(size_t)j * nnz_cap + s];
  }
}
cudaError_t launch_scatter_samples(const float2* samples, const int* idx, const int* nnz, int nnz_cap, int J,
                                   size_t N, float2* y, cudaStream_t s) {
  return launch_k(scatter_samples_kernel, dim3(148 * 4), dim3(256), 0, s, samples, idx, nnz, nnz_cap, J, N, y);
}

// GPU gridding of radial spokes ("initial interpolation of the data to the
// grid"): one thread per (coil, sampled cell); the cell's samples (CSR list built at
// nlinv_plan_set_trajectory[_kb], ascending (spoke, readout) order) are averaged into y_j[cell] --
// plain mean for nearest-cell gridding (R20), Kaiser-Bessel-weighted mean sum h d / sum h with
// the per-entry weights wgt for convolution gridding (R22). Cells off P_k are not written (R16).
__global__ void grid_radial_kernel(const float2* __restrict__ raw, int J, int nraw, const int* __restrict__ cells,
                                   const int* __restrict__ start, const int* __restrict__ sid,
                                   const float* __restrict__ wgt, int nnz, size_t N, float2* __restrict__ y) {
  pdl_wait();
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)J * nnz;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / nnz), e = (int)(t % nnz);
    const int a = start[e], b = start[e + 1];
    float2 acc = make_float2(0.f, 0.f);
    float den = 0.f;
    for (int u = a; u < b; ++u) {
      const float2 v = raw[(size_t)j * nraw + sid[u]];
      const float w = wgt ? wgt[u] : 1.0f;
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
      den += w;
    }
    const float inv = 1.0f / den;
    y[(size_t)j * N + cells[e]] = make_float2(acc.x * inv, acc.y * inv);
  }
}
cudaError_t launch_grid_radial(const float2* raw, int J, int nraw, const int* cells, const int* start, const int* sid,
                               const float* wgt, int nnz, size_t N, float2* y, cudaStream_t s) {
  long long nb = ((long long)J * nnz + 255) / 256;
  if (nb > 148 * 8) nb = 148 * 8;
  if (nb < 1) nb = 1;
  return launch_k(grid_radial_kernel, dim3((unsigned)nb), dim3(256), 0, s, raw, J, nraw, cells, start, sid, wgt, nnz, N,
                  y);
}

cudaError_t launch_init_x(float2* x, long long nrho, long long ntot, cudaStream_t s) {
  return launch_k(init_x_kernel, dim3(vec_grid(ntot)), dim3(kVecThreads), 0, s, x, nrho, ntot);
}

int col_tiles(int ng) {
#define X(L) if (ng == L) return col_tiles_##L();
  NLV_FOR_EACH_NG(X)
#undef X
  return 0;
}

cudaError_t launch_image(int ng, const float2* rho_omega, const float* rss, int nplanes, float2* img, cudaStream_t s) {
  const int Q = (ng / 2) * (ng / 2);
  return launch_k(image_kernel, dim3((Q + 255) / 256), dim3(256), 0, s, rho_omega, rss, nplanes, img, Q);
}
cudaError_t launch_coil_sum(int ng, const float2* S_all, int J, float2* S, cudaStream_t s) {
  const int Q = (ng / 2) * (ng / 2);
  return launch_k(coil_sum_kernel, dim3((Q + 255) / 256), dim3(256), 0, s, S_all, J, S, Q);
}
cudaError_t launch_rss_sum(int ng, const float* rss_all, int J, float* rss, cudaStream_t s) {
  const int Q = (ng / 2) * (ng / 2);
  return launch_k(rss_sum_kernel, dim3((Q + 255) / 256), dim3(256), 0, s, rss_all, J, rss, Q);
}
bool k5cg_fusable(int ng, int J) {
#define X(L) if (ng == L) return k5cg_fusable_##L(J);
  NLV_FOR_EACH_NG(X)
#undef X
  return false;
}
int k5cg_rows(int ng, int J) {
#define X(L) if (ng == L) return k5cg_rows_##L(J);
  NLV_FOR_EACH_NG(X)
#undef X
  return J;
}
bool k234_supported(int ng) {
#define X(L) if (ng == L) return k234_ok_##L();
  NLV_FOR_EACH_NG(X)
#undef X
  return false;
}
cudaError_t launch_k234(int ng, const RowArgs& a, const float2* tw, cudaStream_t s) {
#define X(L) if (ng == L) return launch_k234_##L(a, tw, s);
  NLV_FOR_EACH_NG(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t preload_kernels(int ng) {
  cudaError_t e = cudaErrorInvalidValue;
#define X(L) if (ng == L) e = preload_##L();
  NLV_FOR_EACH_NG(X)
#undef X
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  const void* fs[] = {(const void*)newton_update_kernel, (const void*)r_update_kernel, (const void*)image_kernel,
                      (const void*)coil_sum_kernel, (const void*)rss_sum_kernel, (const void*)xchg_kernel,
                      (const void*)init_x_kernel, (const void*)mask_count_kernel, (const void*)mask_scatter_kernel,
                      (const void*)scatter_samples_kernel, (const void*)grid_radial_kernel};
  for (const void* f : fs)
    if ((e = cudaFuncGetAttributes(&fa, f)) != cudaSuccess) return e;
  return cudaSuccess;
}

int k234_max_clusters(int ng) {
#define X(L) if (ng == L) return k234_max_clusters_##L();
  NLV_FOR_EACH_NG(X)
#undef X
  return -1;
}

}  // namespace nlv
