// Non-templated kernels (rho block, CG vector update, frame output) and the grid-size
// dispatch of the templated FFT-pass kernels (kernels_impl.cuh, one TU per size in inst.cu).
#include "kernels_impl.cuh"

namespace nlv {

// ------------------------------------------------------------------ rho-block kernels
constexpr int kVecThreads = 256;

// Ap_rho = M . S + alpha p_rho (whole grid), <p_rho, Ap_rho> partial
__global__ void __launch_bounds__(kVecThreads) rho_finish_kernel(VecArgs a, int L, int with_dot) {
  __shared__ double red[32];
  const int n = L / 2, q = L / 4;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.nrho; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / L), xx = (int)(i % L);
    float2 s = make_float2(0.f, 0.f);
    if (y >= q && y < q + n && xx >= q && xx < q + n) s = a.S[(size_t)(y - q) * n + (xx - q)];
    const float2 pv = a.p[i];
    const float2 o = make_float2(fmaf(a.alpha, pv.x, s.x), fmaf(a.alpha, pv.y, s.y));
    a.out[i] = o;
    acc += (double)pv.x * o.x + (double)pv.y * o.y;
  }
  if (with_dot) {
    const double vv[1] = {acc};
    const int sl[1] = {SC_PAP_RHO + a.iter};
    grid_finish<1>(vv, a.partials, a.counter, a.scal_w, sl, red);
  }
}

// b_rho = M . S - alpha (rho - rho_ref); r = p = b; <b, b> partial
__global__ void __launch_bounds__(kVecThreads) rho_rhs_kernel(VecArgs a, int L) {
  __shared__ double red[32];
  const int n = L / 2, q = L / 4;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.nrho; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / L), xx = (int)(i % L);
    float2 s = make_float2(0.f, 0.f);
    if (y >= q && y < q + n && xx >= q && xx < q + n) s = a.S[(size_t)(y - q) * n + (xx - q)];
    const float2 d = csub(a.x[i], a.xref[i]);
    const float2 b = make_float2(fmaf(-a.alpha, d.x, s.x), fmaf(-a.alpha, d.y, s.y));
    a.r[i] = b;
    a.p[i] = b;
    acc += (double)b.x * b.x + (double)b.y * b.y;
  }
  const double vv[1] = {acc};
  const int sl[1] = {SC_RR_RHO + 0};
  grid_finish<1>(vv, a.partials, a.counter, a.scal_w, sl, red);
}

// out_rho = M . S (adjoint operator)
__global__ void __launch_bounds__(kVecThreads) rho_adj_kernel(VecArgs a, int L) {
  const int n = L / 2, q = L / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.nrho; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / L), xx = (int)(i % L);
    float2 s = make_float2(0.f, 0.f);
    if (y >= q && y < q + n && xx >= q && xx < q + n) s = a.S[(size_t)(y - q) * n + (xx - q)];
    a.out[i] = s;
  }
}

// CG step: gamma = rr / <p,Ap>; dx += gamma p; r -= gamma Ap; <r,r> (rho, chat partials).
// Last iteration: x += dx + gamma p (the Newton update x_{n+1} = x_n + dx, Eq. 3).
__global__ void __launch_bounds__(kVecThreads) cg_update_kernel(VecArgs a) {
  __shared__ double red[32];
  const float gamma = cg_gamma(a.scal, a.iter);
  double acc_rho = 0.0, acc_chat = 0.0;
  // two complex numbers per thread-iteration (16-byte accesses); ntot is even (N % 16 == 0)
  const long long n2 = a.ntot / 2;
  const float4* p4 = reinterpret_cast<const float4*>(a.p);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const float4 pv = p4[i];
    float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.iter > 0) d = reinterpret_cast<const float4*>(a.dx)[i];
    d.x = fmaf(gamma, pv.x, d.x); d.y = fmaf(gamma, pv.y, d.y);
    d.z = fmaf(gamma, pv.z, d.z); d.w = fmaf(gamma, pv.w, d.w);
    if (a.last) {
      float4 xv = reinterpret_cast<float4*>(a.x)[i];
      xv.x += d.x; xv.y += d.y; xv.z += d.z; xv.w += d.w;
      reinterpret_cast<float4*>(a.x)[i] = xv;
    } else {
      reinterpret_cast<float4*>(a.dx)[i] = d;
      const float4 av = reinterpret_cast<const float4*>(a.Ap)[i];
      float4 rv = reinterpret_cast<float4*>(a.r)[i];
      rv.x = fmaf(-gamma, av.x, rv.x); rv.y = fmaf(-gamma, av.y, rv.y);
      rv.z = fmaf(-gamma, av.z, rv.z); rv.w = fmaf(-gamma, av.w, rv.w);
      reinterpret_cast<float4*>(a.r)[i] = rv;
      const double s = (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
      if (2 * i < a.nrho) acc_rho += s; else acc_chat += s;
    }
  }
  if (!a.last) {
    const double vv[2] = {acc_rho, acc_chat};
    const int sl[2] = {SC_RR_RHO + a.iter + 1, SC_RR_CHAT + a.iter + 1};
    grid_finish<2>(vv, a.partials, a.counter, a.scal_w, sl, red);
  }
}

// frame output: image = crop_Omega(rho) . sqrt(sum_j |c_j|^2)
__global__ void image_kernel(const float2* __restrict__ rho_omega, const float* __restrict__ rss, float2* img, int Q) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += gridDim.x * blockDim.x) {
    const float s = sqrtf(rss[i]);
    img[i] = cscale(rho_omega[i], s);
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
  const long long cap = 148 * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_rho_finish(int ng, const VecArgs& a, int with_dot, cudaStream_t s) {
  rho_finish_kernel<<<vec_grid(a.nrho), kVecThreads, 0, s>>>(a, ng, with_dot);
  return cudaGetLastError();
}
cudaError_t launch_rho_rhs(int ng, const VecArgs& a, cudaStream_t s) {
  rho_rhs_kernel<<<vec_grid(a.nrho), kVecThreads, 0, s>>>(a, ng);
  return cudaGetLastError();
}
cudaError_t launch_rho_adj(int ng, const VecArgs& a, cudaStream_t s) {
  rho_adj_kernel<<<vec_grid(a.nrho), kVecThreads, 0, s>>>(a, ng);
  return cudaGetLastError();
}
cudaError_t launch_cg_update(int /*ng*/, const VecArgs& a, cudaStream_t s) {
  cg_update_kernel<<<vec_grid(a.ntot / 2), kVecThreads, 0, s>>>(a);
  return cudaGetLastError();
}
__global__ void init_x_kernel(float2* x, long long nrho, long long ntot) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ntot; i += (long long)gridDim.x * blockDim.x)
    x[i] = make_float2(i < nrho ? 1.0f : 0.0f, 0.0f);
}
cudaError_t launch_init_x(float2* x, long long nrho, long long ntot, cudaStream_t s) {
  init_x_kernel<<<vec_grid(ntot), kVecThreads, 0, s>>>(x, nrho, ntot);
  return cudaGetLastError();
}

int col_tiles(int ng) {
#define X(L) if (ng == L) return col_tiles_##L();
  NLV_FOR_EACH_NG(X)
#undef X
  return 0;
}

cudaError_t launch_image(int ng, const float2* rho_omega, const float* rss, float2* img, cudaStream_t s) {
  const int Q = (ng / 2) * (ng / 2);
  image_kernel<<<(Q + 255) / 256, 256, 0, s>>>(rho_omega, rss, img, Q);
  return cudaGetLastError();
}

}  // namespace nlv
