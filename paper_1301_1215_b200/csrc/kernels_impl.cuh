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
#include <utility>

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
  // k5cg_kernel: + the r / dx tile (pf) + the CTA's w^-1 columns folded by |k - L/2| (w^-1 is even in k - L/2):
  // (L/2 + 1) x CW floats loaded once before griddepcontrol.wait instead of 2 x L x CW global reads per
  // launch; used where it does not lower the CTAs per SM (2 at <= 115712 B per CTA)
  static constexpr size_t PF0 = SMEM + 64 * sizeof(double) + sizeof(float2) * (size_t)L * CW;
  static constexpr size_t WTAB = sizeof(float) * (size_t)(L / 2 + 1) * CW;
  static constexpr bool kWTab = (PF0 + WTAB <= 115712) || (PF0 > 115712 && PF0 + WTAB <= 232448);
  static constexpr size_t SMEM_PF = PF0 + (kWTab ? WTAB : 0);
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
  template <int L>
  __device__ __forceinline__ float2& first(int i) const { return s[i * CW + c]; }
  // First exchange at CW = 8 (L >= 512): pass 0 stores rows i = (t + T m) R0 + r, so the 4 t-values of
  // a warp are R0 rows apart and hit the same 8-byte banks (2-way conflicts). Rows i and i ^ 1 are
  // swapped when bit log2(R0) of i is set: for the stores that bit is t & 1 and the parity of i is r's,
  // for the loads (i = t + T m + r L / RN) both are bits of t, so the swap is a per-thread row offset
  // folded into the column offset -- no instruction per access.
  static constexpr bool kSwz1(int L) { return CW == 8 && (L == 512 || L == 768 || L == 1024); }
  template <int L>
  __device__ __forceinline__ float2& first_st(int i, int rpar) const {   // rpar = r & 1 (unrolled: constant)
    if constexpr (kSwz1(L)) {
      const int key = (int)(threadIdx.x / CW) & 1;   // t & 1
      return s[i * CW + c + (rpar ? -key : key) * CW];
    } else {
      return s[i * CW + c];
    }
  }
  template <int L>
  __device__ __forceinline__ float2& first_ld(int i) const {
    if constexpr (kSwz1(L)) {
      constexpr int lg = Cfg<L>::R0 == 16 ? 4 : 3;
      const int t = (int)(threadIdx.x / CW);
      const int d = ((t >> lg) & 1) ? ((t & 1) ? -1 : 1) : 0;
      return s[i * CW + c + d * CW];
    } else {
      return s[i * CW + c];
    }
  }
  template <int L>
  __device__ __forceinline__ float2& mid(int i) const { return s[i * CW + c]; }
};
// Row exchange buffer. The first Stockham exchange (buf.first) is XOR-swizzled: slot i lives at
// (i & ~15) | ((i & 15) ^ ((i >> 4) & 15)). The first pass stores at stride R (8 at L = 384, 16 at
// L = 1024), which unswizzled puts a warp's lanes on one or two bank pairs; the swizzle permutes
// within aligned 16-slot blocks, so the reads "t + T m + const" stay conflict-light and cost one
// XOR with a compile-time key. Later exchanges are unswizzled (conflict-light already).
struct RowBuf {
  float2* s;
  __device__ __forceinline__ float2& operator()(int i) const { return s[i]; }
  // first Stockham exchange only (the stride-R stores): the later exchanges are conflict-light
  // unswizzled, and the swizzle's index arithmetic is not free in these issue-bound passes
  template <int L>
  __device__ __forceinline__ float2& first(int i) const { return s[(i & ~15) | ((i & 15) ^ ((i >> 4) & 15))]; }
  template <int L>
  __device__ __forceinline__ float2& first_st(int i, int) const { return first<L>(i); }
  template <int L>
  __device__ __forceinline__ float2& first_ld(int i) const { return first<L>(i); }
  // second exchange (after pass 1, stride NS = R0 stores): unswizzled, the threads t and t + R0 of a
  // row (and the rows sharing a warp) land on the same 8-byte banks at L = 384 / 512 / 768 (2-way
  // conflicts); an XOR of the bit that separates them into bank bit 3 (a full 4-bit key at 512) makes
  // the stores conflict-free and keeps the contiguous reads "t + T m + const" conflict-free
  template <int L>
  __device__ __forceinline__ float2& mid(int i) const {
    if constexpr (L == 384) return s[i ^ (((i >> 4) & 1) << 3)];
    else if constexpr (L == 512) return s[(i & ~15) | ((i & 15) ^ ((i >> 4) & 15))];
    else if constexpr (L == 768) return s[i ^ (((i >> 5) & 1) << 3)];
    else return s[i];
  }
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

// Centred transform without sign flips (R1): for even L with L/2 even,
//   F_c z [k] ∝ (-1)^k FFT((-1)^i z)[k] = FFT(z[. + L/2])[k + L/2],
// and a shift by L/2 of a pass-0 input (last-pass output) index is a compile-time permutation of
// the registers (R0, RL even), so the modulations cost no instructions: load register e from
// index in_idx(t, psh_in(e)), and read position k = out_idx(t, e) from register psh_out(e).
template <int L>
__host__ __device__ constexpr int psh_in(int e) {
  constexpr int R = Cfg<L>::R0;
  return (e / R) * R + (e % R + R / 2) % R;
}
template <int L>
__host__ __device__ constexpr int psh_out(int e) {
  constexpr int R = Sched<L>::RL;
  return (e / R) * R + (e % R + R / 2) % R;
}

// Pass-0 zero masks (fft<..., ZM0>): bit r set if register slots m*R0 + r are structurally zero.
// Omega-row / -column input (half images): positions outside [L/4, 3L/4) are zero.
template <int L>
__host__ __device__ constexpr unsigned omega_in_zmask() {
  unsigned z = 0;
  for (int r = 0; r < Cfg<L>::R0; ++r) {
    const int pos = r * (L / Cfg<L>::R0);
    if (pos < L / 4 || pos >= 3 * L / 4) z |= 1u << r;
  }
  return z;
}
// ... the same input after the half-shift register permutation (psh_in) of the row passes
template <int L>
__host__ __device__ constexpr unsigned omega_shift_zmask() {
  return ((1u << Cfg<L>::R0) - 1u) & ~omega_in_zmask<L>();
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
    __threadfence();  // gpu-scope fence: also invalidates this SM's L1, the partials are read fresh
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      // every thread of the last CTA sums a fixed strided subset, then the fixed block tree
      double acc = 0.0;
      const double* pk = partials + k * kMaxRedBlocks;
      for (unsigned i = threadIdx.x; i < nblk; i += blockDim.x) acc += __ldcg(pk + i);
      const double tot = block_sum(acc, red);
      if (threadIdx.x == 0 && slot[k] >= 0) scal_w[slot[k]] = tot;
    }
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// Grid barrier with one atomic per CTA and no reset: CTA 0 adds 2^31 - (nb - 1), every other CTA
// adds 1, so the word's top bit flips exactly when the last CTA arrives and the low bits return to
// their value (reusable across launches and graph replays). Waiters poll with ld.acquire.gpu.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_sync_flip(unsigned* bar, unsigned nb, bool master) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = master ? (0x80000000u - (nb - 1u)) : 1u;
    __threadfence();   // release: this CTA's writes (ordered before by bar.sync) precede the arrival
    const unsigned old = atomicAdd(bar, inc);
    unsigned spins = 0;
    while (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) == 0u) {
      if (++spins > (1u << 30)) __trap();  // never hang the GPU: abort the context instead
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ peer-memory exchange primitives (f1)
__device__ __forceinline__ unsigned long long* xw_flag(char* w, int k) { return reinterpret_cast<unsigned long long*>(w + 128 * k); }
__device__ __forceinline__ unsigned* xw_counter(char* w, int k) { return reinterpret_cast<unsigned*>(w + 1024 + 128 * k); }
__device__ __forceinline__ double* xw_dots(char* w, int par) { return reinterpret_cast<double*>(w + 2048) + 8 * par; }
__device__ __forceinline__ double* xw_xs(char* w) { return reinterpret_cast<double*>(w + 2304); }
__device__ __forceinline__ float2* xw_S(char* w, int par, size_t Q) { return reinterpret_cast<float2*>(w + kXWinHdr) + (size_t)par * Q; }
__device__ __forceinline__ float* xw_rss(char* w, size_t Q) { return reinterpret_cast<float*>(w + kXWinHdr + 2 * Q * 8); }

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
// this rank's current epoch of kind k (only this rank writes its own flags)
__device__ __forceinline__ unsigned long long x_epoch(const XPeers& xp, int k) {
  return ld_acquire_sys64(xw_flag(xp.win[xp.rank], k));
}
// one thread: publish epoch e of kind k (the data of e are written and fenced by the caller)
__device__ __forceinline__ void x_publish(const XPeers& xp, int k, unsigned long long e) {
  __threadfence_system();
  st_release_sys64(xw_flag(xp.win[xp.rank], k), e);
}
// one thread: wait until every rank published epoch >= e of kind k
__device__ __forceinline__ void x_wait_all(const XPeers& xp, int k, unsigned long long e) {
  for (int h = 0; h < xp.G; ++h) {
    const unsigned long long* f = xw_flag(xp.win[h], k);
    unsigned spins = 0;
    while (ld_acquire_sys64(f) < e) {
      __nanosleep(64);
      if (++spins > (1u << 27)) __trap();   // a peer never arrived: abort the context, never hang
    }
  }
}
// every thread of every CTA: the last CTA of the grid to arrive publishes the next epoch of kind k
// (all CTAs' writes of that epoch's data precede it)
__device__ __forceinline__ void x_publish_last_block(const XPeers& xp, int k) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned nblk = gridDim.x * gridDim.y * gridDim.z;
    const unsigned t = atomicAdd(xw_counter(xp.win[xp.rank], k), 1u);
    s_last = (t == nblk - 1);
    if (s_last) {
      *xw_counter(xp.win[xp.rank], k) = 0u;
      __threadfence();
      x_publish(xp, k, x_epoch(xp, k) + 1);
    }
  }
  __syncthreads();
}
// sum_g S_g[o] over the ranks' published coil-sum planes of epoch e, ascending rank order
__device__ __forceinline__ float2 x_sum_S(const XPeers& xp, unsigned long long e, size_t Q, size_t o) {
  float2 sv = make_float2(0.f, 0.f);
  const int par = (int)(e & 1ull);
  for (int h = 0; h < xp.G; ++h) sv = cadd(sv, xw_S(xp.win[h], par, Q)[o]);
  return sv;
}

// Textbook CG scalars (R9): gamma_i = rr_i / <p_i, A p_i>, beta_i = rr_{i+1} / rr_i.
// rr_i and <p_i, A p_i> are published as (rho, chat) parts; rho is replicated and counted once.
__device__ __forceinline__ double cg_rr(const double* scal, int i) { return scal[SC_RR_RHO + i] + scal[SC_RR_CHAT + i]; }
__device__ __forceinline__ float cg_gamma(const double* scal, int i) {
  const double rr = cg_rr(scal, i);
  const double pap = scal[SC_PAP_RHO + i] + scal[SC_PAP_CHAT + i];
  return rr != 0.0 ? (float)(rr / pap) : 0.0f;
}
__device__ __forceinline__ float cg_beta(const double* scal, int i) {  // beta_i
  const double rr = cg_rr(scal, i);
  return rr != 0.0 ? (float)(cg_rr(scal, i + 1) / rr) : 0.0f;
}

// Single-reduction CG scalars of iteration i (R19): gamma_i = <r_i,r_i>/<p_i,Ap_i> with the direct
// <r_i,r_i>; <r_{i+1},r_{i+1}> by exact expansion (rho and chat parts), beta_i = that / <r_i,r_i>.
__device__ __forceinline__ void cg1_gamma_beta(const double* scal, int i, float* gamma, float* beta) {
  const double rrr = scal[SC_RR_RHO + i], rrc = scal[SC_RR_CHAT + i], rr = rrr + rrc;
  const double pap = scal[SC_PAP_RHO + i] + scal[SC_PAP_CHAT + i];
  const float g = rr != 0.0 ? (float)(rr / pap) : 0.0f;
  const double gd = (double)g;
  const double nr = fmax(rrr - 2.0 * gd * scal[SC_RAP_RHO + i] + gd * gd * scal[SC_AA_RHO + i], 0.0);
  const double nc = fmax(rrc - 2.0 * gd * scal[SC_RAP_CHAT + i] + gd * gd * scal[SC_AA_CHAT + i], 0.0);
  *gamma = g;
  *beta = rr != 0.0 ? (float)((nr + nc) / rr) : 0.0f;
}

// Programmatic dependent launch (PDL): every pass is launched with programmatic stream
// serialisation, so its CTAs are scheduled while the previous pass drains; pdl_wait() blocks
// until the previous grid has completed and its memory is visible, so it must precede every
// read of data produced upstream. pdl_trigger() lets the next pass be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Twiddle table global -> shared with cp.async, so its latency overlaps the pass's own loads;
// the pass waits for it (tw_wait) right before its first transform.
__device__ __forceinline__ void tw_copy_async(float2* tw_s, const float2* tw_g, int L) {
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(tw_s + i);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(tw_g + i));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void tw_wait() {
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
}
// ... while one later commit group (a tile prefetch) may stay in flight
__device__ __forceinline__ void tw_wait_keep1() {
  asm volatile("cp.async.wait_group 1;\n" ::);
  __syncthreads();
}

__device__ __forceinline__ void prefetch_wait() {
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
}

// L2 prefetch of the column tile the CTA one resident wave later will transform (grids of several waves,
// data above L2): the next wave finds its input in L2 while this wave computes. wave = CTAs per resident
// wave (0: off); one prefetch per row segment (threads of column 0).
template <int L>
__device__ __forceinline__ void prefetch_next_wave_cols(const float2* base, size_t plane, int wave, int rlo, int rhi) {
  constexpr int CW = ColGeo<L>::CW;
  if (wave <= 0 || threadIdx.x % CW != 0) return;
  const unsigned nb = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x, nxt = bid + (unsigned)wave;
  if (nxt >= nb) return;
  const float2* d = base + (size_t)(nxt / gridDim.x) * plane + (size_t)(nxt % gridDim.x) * CW;
  for (int r = rlo + (int)(threadIdx.x / CW); r < rhi; r += (int)(blockDim.x / CW))
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(d + (size_t)r * L));
}

// Column-tile prefetch: rows 0..L-1, columns x0..x0+CW-1 of one [L][L] c64 image into shared
// memory laid out [row][CW] (the ColBuf layout: thread (t, c) later reads its rows k at
// dst[k * CW + c]); 16-byte cp.async.cg (L2 only), one commit group.
template <int L, int CW>
__device__ __forceinline__ void tile_prefetch(float2* dst, const float2* img, int x0) {
  constexpr int CPR = CW / 2;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < L * CPR; i += blockDim.x) {
    const int row = i / CPR, c2 = i - row * CPR;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + row * CW + 2 * c2);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(img + (size_t)row * L + x0 + 2 * c2));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// Column-tile prefetch with the tensor memory accelerator: the [L rows][CW columns] tile of coil j
// of a [J][L][L] c64 array, described by a host-built CUtensorMap (3D: x, y, coil; 8-byte elements),
// lands in shared memory as [row][CW] (the ColBuf layout) from ceil(L / 256) box loads issued by one
// thread, completion tracked by an mbarrier (transaction bytes). Replaces L*CW/2 cp.async per CTA.
__device__ __forceinline__ void tma_tile_issue(uint64_t* mbar, float2* dst, const void* tmap, int x0, int j, int L,
                                               int CW) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  const uint32_t bytes = (uint32_t)(L * CW * 8);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
  const int box = L <= 256 ? L : (L % 256 == 0 ? 256 : 192);   // box rows <= 256 (TMA limit)
  for (int y0 = 0; y0 < L; y0 += box) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + (size_t)y0 * CW);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(d), "l"(tmap), "r"(x0), "r"(y0), "r"(j), "r"(mb) : "memory");
  }
}
// the same into an mbarrier already initialised (tma_bar_init) and made visible to the CTA
__device__ __forceinline__ void tma_bar_init(uint64_t* mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tma_tile_issue_ready(uint64_t* mbar, float2* dst, const void* tmap, int x0, int j, int L,
                                                     int CW) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic accesses of dst before the async copy
  const uint32_t bytes = (uint32_t)(L * CW * 8);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
  const int box = L <= 256 ? L : (L % 256 == 0 ? 256 : 192);
  for (int y0 = 0; y0 < L; y0 += box) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + (size_t)y0 * CW);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(d), "l"(tmap), "r"(x0), "r"(y0), "r"(j), "r"(mb) : "memory");
  }
}
__device__ __forceinline__ void tma_tile_wait(uint64_t* mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(mb) : "memory");
  }
}

// debug timeline of one CTA (globaltimer ns), compiled in with -DNLV_TRACE
__device__ __forceinline__ void trace_stamp(unsigned long long* tr, int k) {
#ifdef NLV_TRACE
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[(size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 8 + k] = t;
  }
#endif
}

// ------------------------------------------------------------------ column task (one tile of CW columns)
// Returns this thread's contributions to the (rho, chat) reductions of MODE. The caller owns
// the twiddle table tw (shared) and the exchange buffer xb (shared, L*CW float2). Every thread
// of the CTA must call it (the transform uses __syncthreads).
// PW: real-valued P_k (KB gridding, R22); XP: peer-memory exchange (world > 1) -- separate instantiations,
// so the single-GPU kernels carry none of that code
template <int L, int MODE, bool PW = false, bool XP = false>
__device__ __forceinline__ void col_task(const ColArgs& a, int tile, int j, const float2* tw, float2* xb,
                                         double& acc_rho, double& acc, double* acc3, int rlo = 0, int rhi = L,
                                         bool tw_async = false, const uint32_t* pre_mbits = nullptr) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E, CW = ColGeo<L>::CW;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t N = (size_t)L * L, H = (size_t)n * L, Qs = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;
  constexpr int DIR_FIRST = (MODE == CK_IFFT_W || MODE == CK_IFFT_W_CG || MODE == CK_ADJ1) ? +1 : -1;

  const int tid = threadIdx.x, c = tid % CW, t = tid / CW;
  const int x = tile * CW + c;

  // rho block spread over the coil tiles: tile (j, tile) also handles a contiguous stripe of the
  // N rho elements, so the pass needs no extra CTAs (one wave at 2 CTAs/SM)
  if constexpr (MODE == CK_IFFT_W_CG || MODE == CK_FFT_W_NORMAL || MODE == CK_FFT_W_RHS || MODE == CK_FFT_W_ADJ) {
    {
      constexpr int NTILE = L / CW;
      const int nstripe = a.J * NTILE, stripe = j * NTILE + tile;
      const size_t chunk = (N + nstripe - 1) / nstripe;
      const size_t lo = (size_t)stripe * chunk, hi = (lo + chunk < N) ? lo + chunk : N;
      for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        if constexpr (MODE == CK_IFFT_W_CG) {
          float2 rv = a.rho_r[i];
          const float2 pv = a.rho_p[i];
          if (a.cg1 && a.iter > 0) {
            const float2 av = a.rho_a[i];
            rv = make_float2(fmaf(-a.gamma, av.x, rv.x), fmaf(-a.gamma, av.y, rv.y));
            a.rho_r[i] = rv;
          }
          if (a.iter > 0) {
            const float2 dv = (a.iter > 1) ? a.rho_dx[i] : make_float2(0.f, 0.f);
            a.rho_dx[i] = make_float2(fmaf(a.gamma, pv.x, dv.x), fmaf(a.gamma, pv.y, dv.y));
          }
          a.rho_p[i] = make_float2(fmaf(a.beta, pv.x, rv.x), fmaf(a.beta, pv.y, rv.y));
        } else {
          const int y = (int)(i / L), xx = (int)(i % L);
          float2 sv = make_float2(0.f, 0.f);
          if (xx >= q && xx < q + n && y >= q && y < q + n) {
            const size_t o = (size_t)(y - q) * n + (xx - q);
            if constexpr (XP) sv = x_sum_S(*a.xp, x_epoch(*a.xp, XK_S), Qs, o);   // ranks' planes, rank order
            else for (int sp = 0; sp < a.nS; ++sp) sv = cadd(sv, a.S[sp * Qs + o]);
          }
          if constexpr (MODE == CK_FFT_W_NORMAL) {
            const float2 pv = a.rho_a[i];
            const float2 o = make_float2(fmaf(a.alpha, pv.x, sv.x), fmaf(a.alpha, pv.y, sv.y));
            a.rho_out[i] = o;
            acc_rho += (double)pv.x * o.x + (double)pv.y * o.y;
            if (a.cg1) {
              const float2 rv = a.rho_r[i];
              acc3[0] += (double)rv.x * o.x + (double)rv.y * o.y;
              acc3[1] += (double)o.x * o.x + (double)o.y * o.y;
              acc3[2] += (double)rv.x * rv.x + (double)rv.y * rv.y;
            }
          } else if constexpr (MODE == CK_FFT_W_RHS) {
            const float2 d = csub(a.rho_a[i], a.rho_b[i]);
            const float2 b = make_float2(fmaf(-a.alpha, d.x, sv.x), fmaf(-a.alpha, d.y, sv.y));
            a.rho_r[i] = b;
            a.rho_p[i] = b;
            acc_rho += (double)b.x * b.x + (double)b.y * b.y;
          } else {
            a.rho_out[i] = sv;
          }
        }
      }
    }
  }

  ColBuf<CW> buf{xb, c};
  float2 v[E];

  // ---------------- prologue: pass-0 input pattern, index = row
  if constexpr (MODE == CK_IFFT_W) {
    constexpr int CH = 8;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
      float wv[CH];
      float2 rv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const size_t i = (size_t)S::in_idx(t, e0 + u) * L + x;
        wv[u] = a.winv[i];
        rv[u] = a.src[j * N + i];
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) v[e0 + u] = cscale(rv[u], wv[u] * sgn_of(S::in_idx(t, e0 + u)));
    }
  } else if constexpr (MODE == CK_IFFT_W_CG) {
    // fused CG step: dx += gamma_{i-1} p_{i-1}; p_i = r_i + beta_{i-1} p_{i-1} (iteration 0: p = r)
    constexpr int CH = 8;
    const bool upd = a.iter > 0, hasdx = a.iter > 1;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
      float wv[CH];
      float2 rv[CH], pv[CH], dv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const size_t i = j * N + (size_t)S::in_idx(t, e0 + u) * L + x;
        wv[u] = a.winv[(size_t)S::in_idx(t, e0 + u) * L + x];
        rv[u] = a.r[i];
        pv[u] = a.p[i];
        dv[u] = hasdx ? a.dx[i] : make_float2(0.f, 0.f);
        if (a.cg1 && upd) {   // r_i = r_{i-1} - gamma A p_{i-1} (single-reduction CG, R19)
          const float2 av = a.src2[i];
          rv[u] = make_float2(fmaf(-a.gamma, av.x, rv[u].x), fmaf(-a.gamma, av.y, rv[u].y));
        }
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int yr = S::in_idx(t, e0 + u);
        const size_t i = j * N + (size_t)yr * L + x;
        if (a.cg1 && upd) a.r[i] = rv[u];
        if (upd) a.dx[i] = make_float2(fmaf(a.gamma, pv[u].x, dv[u].x), fmaf(a.gamma, pv[u].y, dv[u].y));
        const float2 sv = make_float2(fmaf(a.beta, pv[u].x, rv[u].x), fmaf(a.beta, pv[u].y, rv[u].y));
        a.p[i] = sv;
        v[e0 + u] = cscale(sv, wv[u] * sgn_of(yr));
      }
    }
  } else if constexpr (MODE == CK_ADJ1) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int yr = S::in_idx(t, e);
      const size_t i = (size_t)yr * L + x;
      const float2 s = a.in[j * N + i];
      if constexpr (PW) v[e] = cscale(cneg_if(s, yr & 1), a.pw[i]);   // real-valued P_k (R22)
      else v[e] = a.mask[i] ? cneg_if(s, yr & 1) : make_float2(0.f, 0.f);
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

  // mask bits of this thread's k-space rows, fetched before the transform (latency hidden)
  uint32_t mbits = 0;
  if constexpr (MODE == CK_PSF || MODE == CK_RESADJ || MODE == CK_FWDP) {
    if (pre_mbits != nullptr) {
      mbits = *pre_mbits;
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) mbits |= (a.mask[(size_t)S::out_idx(t, e) * L + x] ? 1u : 0u) << e;
    }
  }

  if (tw_async) tw_wait();
  trace_stamp(a.trace, 1);
  // half-image input modes: the rows outside Omega are zero (pass-0 pruning)
  constexpr bool kHalfIn = !(MODE == CK_IFFT_W || MODE == CK_IFFT_W_CG || MODE == CK_ADJ1);
  fft<L, DIR_FIRST, kHalfIn ? omega_in_zmask<L>() : 0u>(v, t, tw, buf, SyncBlock{});
  trace_stamp(a.trace, 2);

  // ---------------- middle: k-space pointwise (registers hold output pattern, index = k)
  if constexpr (MODE == CK_PSF || MODE == CK_RESADJ) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      const bool m = (mbits >> e) & 1u;
      if constexpr (PW) {   // real-valued P_k = sqrt(PSF) (R22): P_k^2 in the PSF pass
        const float w = m ? a.pw[(size_t)k * L + x] : 0.f;
        if constexpr (MODE == CK_PSF) {
          v[e] = cscale(v[e], w * w);
        } else {
          // r = P (y - F_c x): the IFFT consumes (-1)^k P r = P^2 ((-1)^k y - G), ||r||^2 = sum P^2 |.|^2
          float2 d = make_float2(0.f, 0.f);
          if (m) {
            d = csub(cneg_if(a.y[j * N + (size_t)k * L + x], k & 1), v[e]);
            const float w2 = w * w;
            acc += (double)w2 * ((double)d.x * d.x + (double)d.y * d.y);
            d = cscale(d, w2);
          }
          v[e] = d;
        }
      } else if constexpr (MODE == CK_PSF) {
        // (-1)^k post-sign of the FFT and pre-sign of the IFFT cancel
        v[e] = m ? v[e] : make_float2(0.f, 0.f);
      } else {
        // r = P (y - F x), F x = (-1)^k G; the IFFT consumes (-1)^k r = P((-1)^k y - G)
        float2 rr = make_float2(0.f, 0.f);
        if (m) {
          const float2 yv = cneg_if(a.y[j * N + (size_t)k * L + x], k & 1);
          rr = csub(yv, v[e]);
          acc += (double)rr.x * rr.x + (double)rr.y * rr.y;
        }
        v[e] = rr;
      }
    }
    out_to_in<L>(v, t, buf, SyncBlock{});
    trace_stamp(a.trace, 3);
    fft<L, +1>(v, t, tw, buf, SyncBlock{});
    trace_stamp(a.trace, 4);
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
      const bool m = (mbits >> e) & 1u;
      if constexpr (PW)
        a.out[j * N + (size_t)k * L + x] = m ? cscale(cneg_if(v[e], k & 1), a.pw[(size_t)k * L + x]) : make_float2(0.f, 0.f);
      else
        a.out[j * N + (size_t)k * L + x] = m ? cneg_if(v[e], k & 1) : make_float2(0.f, 0.f);
    }
  } else {  // CK_FFT_W_*: operands loaded in chunks so each chunk's loads are in flight together
    constexpr int CH = 8;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
      float wv[CH];
      float2 o1[CH], o2[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const size_t i = (size_t)S::out_idx(t, e0 + u) * L + x;
        wv[u] = a.winv[i];
        if constexpr (MODE == CK_FFT_W_NORMAL) {
          o1[u] = a.src2[j * N + i];
          if (a.cg1) o2[u] = a.r[j * N + i];
        }
        if constexpr (MODE == CK_FFT_W_RHS) {
          o1[u] = a.src[j * N + i];
          o2[u] = a.src2[j * N + i];
        }
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int k = S::out_idx(t, e0 + u);
        const size_t i = (size_t)k * L + x;
        const float2 val = cscale(v[e0 + u], wv[u] * sgn_of(k));
        if constexpr (MODE == CK_FFT_W_NORMAL) {
          const float2 pv = o1[u];
          const float2 o = make_float2(fmaf(a.alpha, pv.x, val.x), fmaf(a.alpha, pv.y, val.y));
          a.out[j * N + i] = o;
          acc += (double)pv.x * o.x + (double)pv.y * o.y;
          if (a.cg1) {
            const float2 rv = o2[u];
            acc3[3] += (double)rv.x * o.x + (double)rv.y * o.y;
            acc3[4] += (double)o.x * o.x + (double)o.y * o.y;
            acc3[5] += (double)rv.x * rv.x + (double)rv.y * rv.y;
          }
        } else if constexpr (MODE == CK_FFT_W_RHS) {
          const float2 d = csub(o1[u], o2[u]);
          const float2 b = make_float2(fmaf(-a.alpha, d.x, val.x), fmaf(-a.alpha, d.y, val.y));
          a.r[j * N + i] = b;
          a.p[j * N + i] = b;
          v[e0 + u] = b;   // kept for the fused K1 of iteration 0
          acc += (double)b.x * b.x + (double)b.y * b.y;
        } else {
          a.out[j * N + i] = val;
        }
      }
    }
  }
  // Newton rhs fused with K1 of CG iteration 0 (p_0 = r_0 = b): t = w^-1 b -> column IFFT
  if constexpr (MODE == CK_FFT_W_RHS) {
    if (a.fuse_k1) {
      constexpr int CH = 8;
#pragma unroll
      for (int e0 = 0; e0 < E; e0 += CH) {
        float wv[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) wv[u] = a.winv[(size_t)S::out_idx(t, e0 + u) * L + x];
#pragma unroll
        for (int u = 0; u < CH; ++u) v[e0 + u] = cscale(v[e0 + u], wv[u] * sgn_of(S::out_idx(t, e0 + u)));
      }
      out_to_in<L>(v, t, buf, SyncBlock{});
      fft<L, +1>(v, t, tw, buf, SyncBlock{});
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (out_is_omega<L>(e)) {
          const int k = S::out_idx(t, e);
          a.t1[j * H + (size_t)(k - q) * L + x] = cscale(v[e], invL * sgn_of(k));
        }
      }
    }
  }
}

#ifndef NLV_MINB
#define NLV_MINB 2  // <= 128 registers: two 256-thread CTAs per SM (more registers halve residency)
#endif
// PW, XP: see col_task. CG1: the single-reduction CG flag (K1 and K5 of the unfused CG) as a compile-time
// constant, so each instantiation holds only the code its launches run
template <int L, int MODE, bool PW = false, bool XP = false, bool CG1 = false, bool FK1 = false>
__global__ void __launch_bounds__(ColGeo<L>::THREADS, NLV_MINB) col_kernel(ColArgs a, const float2* __restrict__ twg) {
  a.cg1 = CG1 ? 1 : 0;
  if constexpr (MODE == CK_FFT_W_RHS) a.fuse_k1 = FK1 ? 1 : 0;   // the Newton rhs fused with K1 (FK1)
  constexpr int CW = ColGeo<L>::CW;
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  double* red = reinterpret_cast<double*>(xb + (size_t)L * CW);
  trace_stamp(a.trace, 0);
  tw_copy_async(tw, twg, L);
  // K3: P_k is fixed for the frame (set before its first pass): its bits are read (L2-coherent
  // ld.global.cg) before griddepcontrol.wait
  uint32_t mb = 0;
  if constexpr (MODE == CK_PSF) {
    using S = Sched<L>;
    const int c = threadIdx.x % CW, t = threadIdx.x / CW, x = blockIdx.x * CW + c;
#pragma unroll
    for (int e = 0; e < Cfg<L>::E; ++e) mb |= (__ldcg(a.mask + (size_t)S::out_idx(t, e) * L + x) ? 1u : 0u) << e;
  }
  pdl_wait();
  pdl_trigger();
  if constexpr (XP && (MODE == CK_FFT_W_NORMAL || MODE == CK_FFT_W_RHS || MODE == CK_FFT_W_ADJ)) {
    // peer exchange: every rank's K4 has published its coil-sum plane
    if (threadIdx.x == 0) x_wait_all(*a.xp, XK_S, x_epoch(*a.xp, XK_S));
    __syncthreads();
  }
  if constexpr (MODE == CK_IFFT_W_CG) {
    if (a.cg1) {
      if (a.iter > 0) cg1_gamma_beta(a.scal, a.iter - 1, &a.gamma, &a.beta);
      else a.gamma = a.beta = 0.0f;
    } else {
      a.gamma = (a.iter > 0) ? cg_gamma(a.scal, a.iter - 1) : 0.0f;
      a.beta = (a.iter > 0) ? cg_beta(a.scal, a.iter - 1) : 0.0f;
    }
  }
  double acc_rho = 0.0, acc = 0.0;
  const int j = (int)blockIdx.y;
  double acc3[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};   // single-reduction CG dots (rho: 0-2, chat: 3-5)
  col_task<L, MODE, PW, XP>(a, blockIdx.x, j, tw, xb, acc_rho, acc, acc3, 0, L, true, MODE == CK_PSF ? &mb : nullptr);
  trace_stamp(a.trace, 5);
  if constexpr (MODE == CK_RESADJ || MODE == CK_FFT_W_RHS || MODE == CK_FFT_W_NORMAL) {
    if (MODE == CK_FFT_W_NORMAL && a.cg1 && a.partials != nullptr) {
      const double vv[8] = {acc_rho, acc, acc3[0], acc3[3], acc3[1], acc3[4], acc3[2], acc3[5]};
      const int sl[8] = {SC_PAP_RHO + a.iter, SC_PAP_CHAT + a.iter, SC_RAP_RHO + a.iter, SC_RAP_CHAT + a.iter,
                         SC_AA_RHO + a.iter,  SC_AA_CHAT + a.iter,  SC_RR_RHO + a.iter,  SC_RR_CHAT + a.iter};
      grid_finish<8>(vv, a.partials, a.counter, a.scal_w, sl, red);
    } else if (a.partials != nullptr) {
      const double vv[2] = {acc_rho, acc};
      const int sl[2] = {a.out_slot_rho, a.out_slot};
      grid_finish<2>(vv, a.partials, a.counter, a.scal_w, sl, red);
    }
  }
  trace_stamp(a.trace, 6);
}


// ------------------------------------------------------------------ fused K5 + CG + K1, one grid barrier
// One CG iteration's tail (P:233 CG) as one cooperative pass with a SINGLE grid
// barrier: K5 (column FFT -> A p = w^-1 . + alpha p) and, before the barrier, the block dots
// <p,Ap>, <r,r>, <r,Ap>, <Ap,Ap> (rho and chat parts). After the barrier every CTA forms, in the
// same fixed order,
//   gamma_i = <r_i,r_i> / <p_i,Ap_i>,   <r_i,r_i> of the stored r_i, computed in this pass
//   <r_{i+1},r_{i+1}> = <r_i,r_i> - 2 gamma_i Re<r_i,Ap_i> + gamma_i^2 <Ap_i,Ap_i>   (R19)
//   beta_i = <r_{i+1},r_{i+1}> / <r_i,r_i>
// and runs r -= gamma Ap, dx += gamma p, p = r + beta p and K1 of iteration i+1 (w^-1 p -> column
// IFFT -> T1) on its tile; the last iteration does the Newton update x += dx + gamma p instead.
// r (or dx) is prefetched into shared memory while the K5 transform runs; p is parked in the
// exchange buffer. The textbook form needs a second barrier for <r_{i+1}, r_{i+1}> (R19). <r_i,r_i>
// must be the directly computed one: feeding the expanded value back into the next expansion
// accumulates its absolute error and ruins late iterations (measured in an fp32 model: 5e-2 on
// the C1 image vs 6e-5 with the direct <r_i,r_i>).
template <int L, bool XP, bool LAST, bool TM>
__device__ __forceinline__ void k5cg_task(const ColArgs& a, const float2* tw, float2* xb, float2* pf, double* red,
                                          const float* wt) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int E = C::E, CW = ColGeo<L>::CW;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t N = (size_t)L * L, H = (size_t)n * L, Qs = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;
  constexpr int NV = 8;   // pAp, rAp, ApAp, rr; each (rho, chat)
  const int tid = threadIdx.x, c = tid % CW, t = tid / CW;
  const int tile = blockIdx.x, j = blockIdx.y;
  const int x = tile * CW + c;
  // CTA rows j >= J carry no coil tile, only their stripe of the rho block: with few local coils (a
  // coil-sharded rank) the N-element rho stripe work would otherwise fall on 24 J CTAs (k5cg_rows)
  const bool tcta = j < a.J;
  // the last CG iteration (Newton update) and the others are separate instantiations: each launch's
  // code is one path only (the kernel is large; smaller per-launch code means fewer instruction misses)
  constexpr bool last = LAST;
  const bool hasdx = a.iter > 0;
  const unsigned nb = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  ColBuf<CW> buf{xb, c};
  // w^-1 at k-space row k of this thread's column (global index i): the folded shared table or global memory
  // Register e holds k = t + out_off(e); when T divides L/2 and every offset, k - L/2 has the sign of
  // out_off(e) - L/2 for all t, so the table row is +-t + a compile-time constant (two base pointers)
  constexpr bool kFold = ((L / 2) % C::T == 0) && ((L / S::RL) % C::T == 0);
  const float* wpos = wt + t * CW + c;
  const float* wneg = wt - t * CW + c;
  auto w_at = [&](int e, int k, size_t i) -> float {
    if constexpr (ColGeo<L>::kWTab && kFold) {
      const int o = S::out_off(e);
      return (o >= L / 2) ? wpos[(o - L / 2) * CW] : wneg[(L / 2 - o) * CW];
    } else if constexpr (ColGeo<L>::kWTab) {
      const int r = k >= L / 2 ? k - L / 2 : L / 2 - k;
      return wt[r * CW + c];
    } else {
      return a.winv[i];
    }
  };

  // r (dx in the last iteration) was written by the previous CG iteration's pass, which completed
  // before the passes in between could run: the L2-only (cp.async.cg) prefetch is issued before
  // griddepcontrol.wait and overlaps the drain of the previous pass
  bool pf_on = false, pf_tma = false;
  __shared__ alignas(8) uint64_t pf_bar;
  // p tile by TMA into the exchange buffer once the column FFT no longer needs it (p is parked there)
  __shared__ alignas(8) uint64_t pp_bar;
  // TM: the TMA tensor maps exist (default; NLINV_TMA=0 builds the plan without them) -- a template
  // parameter, so the p-tile branches of the per-element loops fold away
  const bool p_tma = TM && tcta;
  if (p_tma && tid == 0) tma_bar_init(&pp_bar);   // visible to the CTA at the FFT's first block barrier
  const void* tmap = last ? a.tmap_dx : a.tmap_r;
  if (!tcta) {
    // rho-only CTA: no tile prefetch
  } else if (TM && (!last || hasdx)) {   // TMA (UTMALDG): one thread issues the tile loads
    if (tid == 0) tma_tile_issue(&pf_bar, pf, tmap, tile * CW, j, L, CW);
    pf_tma = true;
  } else if (!TM && !last) {
    tile_prefetch<L, CW>(pf, a.r + j * N, tile * CW);
    pf_on = true;
  } else if (!TM && hasdx) {
    tile_prefetch<L, CW>(pf, a.dx + j * N, tile * CW);
    pf_on = true;
  }
  pdl_wait();
  pdl_trigger();
  // peer exchange: wait for every rank's coil-sum plane of this iteration (published by its K4)
  unsigned long long eS = 0, eD = 0;
  if constexpr (XP) {
    eS = x_epoch(*a.xp, XK_S);
    eD = x_epoch(*a.xp, XK_DOTS) + 1;   // read before CTA 0 publishes it (after the grid barrier)
    if (tid == 0) x_wait_all(*a.xp, XK_S, eS);
    __syncthreads();
  }

  // prologue: T4 (Omega rows only; the others are zero)
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (in_is_omega<L>(e) && tcta) {
      const int yr = S::in_idx(t, e);
      v[e] = cneg_if(a.in[j * H + (size_t)(yr - q) * L + x], yr & 1);
    } else {
      v[e] = make_float2(0.f, 0.f);
    }
  }

  // rho block stripe of this tile: A p_rho = M sum_s S_s + alpha p_rho (replicated rho).
  // Dot partials in fp64 per term: fp32 products underflow once CG has driven r, p to ~1e-20
  // (the first Newton step from rho = 1, chat = 0 reaches ||r|| ~ 1e-30), giving 0/0.
  double d[NV] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int nstripe = (int)nb, stripe = (int)bid;   // one stripe per CTA (tile and rho-only CTAs)
  const size_t chunk = (N + nstripe - 1) / nstripe;
  const size_t lo = (size_t)stripe * chunk, hi = (lo + chunk < N) ? lo + chunk : N;
  // stripe values stay in registers when the stripe is <= SR elements per thread (C2: 2); the
  // loads of all SR elements are issued together
  constexpr int SR = 2;
  const bool sreg = (hi - lo) <= (size_t)SR * blockDim.x;
  float2 so[SR], sp[SR], sr[SR];
  auto stripe_sum = [&](size_t i) {
    const int y = (int)(i / L), xx = (int)(i % L);
    float2 sv = make_float2(0.f, 0.f);
    if (xx >= q && xx < q + n && y >= q && y < q + n) {
      const size_t o = (size_t)(y - q) * n + (xx - q);
      if constexpr (XP) sv = x_sum_S(*a.xp, eS, Qs, o);   // the ranks' coil-sum planes, rank order
      else for (int s2 = 0; s2 < a.nS; ++s2) sv = cadd(sv, a.S[s2 * Qs + o]);
    }
    return sv;
  };
  if (sreg) {
    float2 sv[SR];
#pragma unroll
    for (int u = 0; u < SR; ++u) {
      const size_t i = lo + tid + (size_t)u * blockDim.x;
      const bool ok = i < hi;
      sp[u] = ok ? a.rho_a[i] : make_float2(0.f, 0.f);
      sr[u] = (ok && !last) ? a.rho_r[i] : make_float2(0.f, 0.f);
      sv[u] = ok ? stripe_sum(i) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < SR; ++u) {
      const float2 pv = sp[u], rv = sr[u];
      const float2 o = make_float2(fmaf(a.alpha, pv.x, sv[u].x), fmaf(a.alpha, pv.y, sv[u].y));
      so[u] = o;
      d[0] += (double)pv.x * o.x + (double)pv.y * o.y;
      d[2] += (double)rv.x * o.x + (double)rv.y * o.y;
      d[4] += (double)o.x * o.x + (double)o.y * o.y;
      d[6] += (double)rv.x * rv.x + (double)rv.y * rv.y;
    }
  } else {
    for (size_t i = lo + tid; i < hi; i += blockDim.x) {
      const float2 sv = stripe_sum(i);
      const float2 pv = a.rho_a[i];
      const float2 o = make_float2(fmaf(a.alpha, pv.x, sv.x), fmaf(a.alpha, pv.y, sv.y));
      a.rho_out[i] = o;
      d[0] += (double)pv.x * o.x + (double)pv.y * o.y;
      if (!last) {
        const float2 rv = a.rho_r[i];
        d[6] += (double)rv.x * rv.x + (double)rv.y * rv.y;
        d[2] += (double)rv.x * o.x + (double)rv.y * o.y;
        d[4] += (double)o.x * o.x + (double)o.y * o.y;
      }
    }
  }

  if (pf_on) tw_wait_keep1();
  else tw_wait();
  trace_stamp(a.trace, 1);
  if (tcta)
    fft<L, -1, omega_in_zmask<L>()>(v, t, tw, buf, SyncBlock{}, [&] {   // T4: Omega rows only
      if (p_tma && tid == 0) tma_tile_issue_ready(&pp_bar, xb, a.tmap_p, tile * CW, j, L, CW);
    });
  trace_stamp(a.trace, 2);
  if (pf_on) prefetch_wait();   // the r / dx tile is complete (all threads' copies)
  if (pf_tma) tma_tile_wait(&pf_bar);
  if (p_tma) tma_tile_wait(&pp_bar);

  // epilogue: A p_chat = w^-1 (-1)^k . + alpha p; p parked in the (now free) exchange buffer
  if (tcta) {
    constexpr int CH = 8;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
      float wv[CH];
      float2 pv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const size_t i = (size_t)S::out_idx(t, e0 + u) * L + x;
        wv[u] = w_at(e0 + u, S::out_idx(t, e0 + u), i);
        pv[u] = p_tma ? buf(S::out_idx(t, e0 + u)) : a.p[j * N + i];
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int k = S::out_idx(t, e0 + u);
        const float2 val = cscale(v[e0 + u], wv[u] * sgn_of(k));
        const float2 o = make_float2(fmaf(a.alpha, pv[u].x, val.x), fmaf(a.alpha, pv[u].y, val.y));
        v[e0 + u] = o;
        if (!p_tma) buf(k) = pv[u];
        d[1] += (double)pv[u].x * o.x + (double)pv[u].y * o.y;
        // <r_i, r_i> directly from the stored r_i (R19); the last iteration takes the previous
        // pass's partials of the r_i it wrote (rr_next below) instead of reading r again
        if (!last) {
          const float2 rv = pf[k * CW + c];
          d[7] += (double)rv.x * rv.x + (double)rv.y * rv.y;
          d[3] += (double)rv.x * o.x + (double)rv.y * o.y;
          d[5] += (double)o.x * o.x + (double)o.y * o.y;
        }
      }
    }
  }
  trace_stamp(a.trace, 7);

  // block partials (warp trees, then warps in index order) -> fpart[k][bid]; grid barrier
  {
    const int w = tid >> 5, lane = tid & 31, nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double vk = d[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) vk += __shfl_xor_sync(0xffffffffu, vk, o);
      if (lane == 0) red[8 + w * NV + k] = vk;
    }
    __syncthreads();
    if (tid < NV) {
      double sk = 0.0;
      for (int ww = 0; ww < nw; ++ww) sk += red[8 + ww * NV + tid];
      a.fpart[tid * nb + bid] = sk;
    }
    grid_sync_flip(a.bar_count, nb, bid == 0);
    trace_stamp(a.trace, 3);
    // totals: warp w sums value k = w (+ nw ...) over all CTAs in a fixed order -> identical in every CTA
    for (int k = w; k < NV; k += nw) {
      double sk = 0.0;
      // the partials of 8 CTAs per lane are loaded together (independent L2 loads in flight), then
      // added in ascending CTA order, the same order in every CTA
      for (unsigned b0 = lane; b0 < nb; b0 += 256) {
        double tk[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tk[u] = (b0 + 32u * u < nb) ? __ldcg(a.fpart + k * nb + b0 + 32u * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) sk += tk[u];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sk += __shfl_xor_sync(0xffffffffu, sk, o);
      if (lane == 0) red[k] = sk;
    }
    __syncthreads();
    if (last) {
      // <r_{L-1}, r_{L-1}> of the stored r: summed by the previous fused pass as it wrote r (per-CTA
      // partials in fpart[8 nb ..], same CTA grid, fixed order), or the rhs pass's <b, b> when L = 1
      if (w == 0) {
        double sr = 0.0, sc = 0.0;
        if (a.iter > 0) {
          for (unsigned b0 = lane; b0 < nb; b0 += 256) {
            double tr[8], tc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const bool ok = b0 + 32u * u < nb;
              tr[u] = ok ? __ldcg(a.fpart + 8 * nb + b0 + 32u * u) : 0.0;
              tc[u] = ok ? __ldcg(a.fpart + 9 * nb + b0 + 32u * u) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              sr += tr[u];
              sc += tc[u];
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, o);
            sc += __shfl_xor_sync(0xffffffffu, sc, o);
          }
        } else {
          sr = a.scal[SC_RR_RHO];
          sc = a.scal[SC_RR_CHAT];
        }
        if (lane == 0) {
          red[6] = sr;
          red[7] = sc;
        }
      }
      __syncthreads();
    }
  }
  if constexpr (XP) {
    // peer exchange of the dots (one epoch of kind XK_DOTS): CTA 0 publishes this rank's totals; every
    // CTA waits for all ranks and forms the global totals in the same order on every rank: the chat
    // parts summed over ranks (ascending), the replicated rho parts taken from rank 0, so gamma and
    // beta -- and with them the rho replicas -- are bit-identical on all ranks
    if (bid == 0 && tid == 0) {
      double* dd = xw_dots(a.xp->win[a.xp->rank], (int)(eD & 1ull));
      for (int k = 0; k < NV; ++k) dd[k] = red[k];
      x_publish(*a.xp, XK_DOTS, eD);
    }
    if (tid == 0) x_wait_all(*a.xp, XK_DOTS, eD);
    __syncthreads();
    double gk = 0.0;
    if (tid < NV) {
      const int par = (int)(eD & 1ull);
      if ((tid & 1) == 0) {
        gk = __ldcv(xw_dots(a.xp->win[0], par) + tid);
      } else {
        for (int h = 0; h < a.xp->G; ++h) gk += __ldcv(xw_dots(a.xp->win[h], par) + tid);
      }
    }
    __syncthreads();
    if (tid < NV) red[tid] = gk;
    __syncthreads();
  }
  // <r_i, r_i>: computed in this pass from the stored r_i (R19)
  trace_stamp(a.trace, 5);   // post-barrier totals done
  const double rr_r = red[6];
  const double rr_c = red[7];
  const double rr = rr_r + rr_c;
  const double pap = red[0] + red[1];
  const float gamma = (rr != 0.0) ? (float)(rr / pap) : 0.0f;
  float beta = 0.0f;
  if (!last) {
    const double g = (double)gamma;
    const double nr = fmax(rr_r - 2.0 * g * red[2] + g * g * red[4], 0.0);
    const double nc = fmax(rr_c - 2.0 * g * red[3] + g * g * red[5], 0.0);
    beta = (rr != 0.0) ? (float)((nr + nc) / rr) : 0.0f;
  }
  if (bid == 0 && tid == 0) {   // the direct <r_i, r_i> (the next pass overwrites slot i + 1 with its own)
    a.scal_w[SC_RR_RHO + a.iter] = rr_r;
    a.scal_w[SC_RR_CHAT + a.iter] = rr_c;
  }
  if (bid == 0 && tid == 0) {
    a.scal_w[SC_PAP_RHO + a.iter] = red[0];
    a.scal_w[SC_PAP_CHAT + a.iter] = red[1];
  }

  if (last) {
    // Newton update x_{n+1} = x_n + dx + gamma_{L-1} p_{L-1} (Eq. 3) on this tile and stripe
    if (tcta) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        const size_t i = j * N + (size_t)k * L + x;
        const float2 pv = buf(k);
        const float2 dv = hasdx ? pf[k * CW + c] : make_float2(0.f, 0.f);
        float2 xv = a.xc[i];
        xv.x += fmaf(gamma, pv.x, dv.x);
        xv.y += fmaf(gamma, pv.y, dv.y);
        a.xc[i] = xv;
        // the next set point's column pass (CK_IFFT_W) folded in: w^-1 x_{n+1} of this tile -> T1 below
        v[e] = cscale(xv, w_at(e, k, (size_t)k * L + x) * sgn_of(k));
      }
    }
    auto newton_rho = [&](size_t i, float2 pv) {
      const float2 dv = hasdx ? a.rho_dx[i] : make_float2(0.f, 0.f);
      float2 xv = a.x_rho[i];
      xv.x += fmaf(gamma, pv.x, dv.x);
      xv.y += fmaf(gamma, pv.y, dv.y);
      a.x_rho[i] = xv;
    };
    if (sreg) {
#pragma unroll
      for (int u = 0; u < SR; ++u) {
        const size_t i = lo + tid + (size_t)u * blockDim.x;
        if (i < hi) newton_rho(i, sp[u]);
      }
    } else {
      for (size_t i = lo + tid; i < hi; i += blockDim.x) newton_rho(i, a.rho_a[i]);
    }
    if (!a.fold_sp) return;
    // column IFFT of w^-1 x_{n+1} restricted to the Omega rows, into T1: what the next Newton step's set
    // point (or the frame's RSS image) would compute in its own column pass
    __syncthreads();   // every parked p has been read: xb becomes the exchange buffer again
    if (!tcta) return;
    out_to_in<L>(v, t, buf, SyncBlock{});
    fft<L, +1>(v, t, tw, buf, SyncBlock{});
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        a.t1[j * H + (size_t)(k - q) * L + x] = cscale(v[e], invL * sgn_of(k));
      }
    }
    return;
  }

  // r_{i+1} = r - gamma Ap; dx += gamma p; p_{i+1} = r_{i+1} + beta p (in place); t = w^-1 p_{i+1}
  // (K1 prologue). <r_{i+1}, r_{i+1}> partials of the stored r_{i+1} for the last iteration (rr_next)
  double rrn_r = 0.0, rrn_c = 0.0;
  if (tcta) {
    constexpr int CH = 8;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
      float wv[CH];
      float2 dv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const size_t ii = (size_t)S::out_idx(t, e0 + u) * L + x;
        wv[u] = w_at(e0 + u, S::out_idx(t, e0 + u), ii);
        dv[u] = hasdx ? a.dx[j * N + ii] : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int k = S::out_idx(t, e0 + u);
        const size_t i = j * N + (size_t)k * L + x;
        const float2 rv = pf[k * CW + c], pv = buf(k);
        const float2 rn = make_float2(fmaf(-gamma, v[e0 + u].x, rv.x), fmaf(-gamma, v[e0 + u].y, rv.y));
        a.r[i] = rn;
        rrn_c += (double)rn.x * rn.x + (double)rn.y * rn.y;
        a.dx[i] = make_float2(fmaf(gamma, pv.x, dv[u].x), fmaf(gamma, pv.y, dv[u].y));
        const float2 pn = make_float2(fmaf(beta, pv.x, rn.x), fmaf(beta, pv.y, rn.y));
        a.p[i] = pn;
        v[e0 + u] = cscale(pn, wv[u] * sgn_of(k));
      }
    }
  }
  trace_stamp(a.trace, 6);   // coil-tile updates issued
  auto update_rho = [&](size_t i, float2 av, float2 rv, float2 pv) {
    const float2 rn = make_float2(fmaf(-gamma, av.x, rv.x), fmaf(-gamma, av.y, rv.y));
    a.rho_r[i] = rn;
    rrn_r += (double)rn.x * rn.x + (double)rn.y * rn.y;
    const float2 dv = hasdx ? a.rho_dx[i] : make_float2(0.f, 0.f);
    a.rho_dx[i] = make_float2(fmaf(gamma, pv.x, dv.x), fmaf(gamma, pv.y, dv.y));
    a.rho_p[i] = make_float2(fmaf(beta, pv.x, rn.x), fmaf(beta, pv.y, rn.y));
  };
  if (sreg) {
#pragma unroll
    for (int u = 0; u < SR; ++u) {
      const size_t i = lo + tid + (size_t)u * blockDim.x;
      if (i < hi) update_rho(i, so[u], sr[u], sp[u]);
    }
  } else {
    for (size_t i = lo + tid; i < hi; i += blockDim.x) update_rho(i, a.rho_out[i], a.rho_r[i], a.rho_a[i]);
  }
  trace_stamp(a.trace, 4);
  {  // <r_{i+1}, r_{i+1}> partials of this CTA (warp trees, warps in order) for the next pass
    const int w = tid >> 5, lane = tid & 31, nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rrn_r += __shfl_xor_sync(0xffffffffu, rrn_r, o);
      rrn_c += __shfl_xor_sync(0xffffffffu, rrn_c, o);
    }
    if (lane == 0) {
      red[8 + 2 * w] = rrn_r;
      red[9 + 2 * w] = rrn_c;
    }
    __syncthreads();
    if (tid == 0) {
      double sr = 0.0, sc = 0.0;
      for (int ww = 0; ww < nw; ++ww) {
        sr += red[8 + 2 * ww];
        sc += red[9 + 2 * ww];
      }
      a.fpart[8 * nb + bid] = sr;
      a.fpart[9 * nb + bid] = sc;
    }
  }
  __syncthreads();   // every parked p has been read: xb becomes the exchange buffer again
  if (!tcta) return;
  out_to_in<L>(v, t, buf, SyncBlock{});
  fft<L, +1>(v, t, tw, buf, SyncBlock{});
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (out_is_omega<L>(e)) {
      const int k = S::out_idx(t, e);
      a.t1[j * H + (size_t)(k - q) * L + x] = cscale(v[e], invL * sgn_of(k));
    }
  }
}

template <int L, bool XP, bool LAST = false, bool TM = true>
__global__ void __launch_bounds__(ColGeo<L>::THREADS, NLV_MINB) k5cg_kernel(ColArgs a, const float2* __restrict__ twg) {
  constexpr int CW = ColGeo<L>::CW;
  extern __shared__ __align__(128) float4 smem_raw[];   // pf (TMA destination) is 128-byte aligned
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  double* red = reinterpret_cast<double*>(xb + (size_t)L * CW);   // 128 doubles
  float2* pf = reinterpret_cast<float2*>(red + 128);
  float* wt = reinterpret_cast<float*>(pf + (size_t)L * CW);
  trace_stamp(a.trace, 0);
  if constexpr (ColGeo<L>::kWTab) {
    // w^-1 is fixed for the plan: its folded columns join the twiddles' cp.async group, before the wait.
    // Row r of the table = |k - L/2| = r, read from global row L/2 + r (row 0 for r = L/2)
    constexpr int C4 = CW / 4;   // 16-byte chunks per row
    const int x0 = blockIdx.x * CW;
    for (int i = threadIdx.x; i < (L / 2 + 1) * C4; i += blockDim.x) {
      const int r = i / C4, c4 = i - r * C4;
      const int gy = (r == L / 2) ? 0 : L / 2 + r;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(wt + r * CW + 4 * c4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(a.winv + (size_t)gy * L + x0 + 4 * c4));
    }
  }
  tw_copy_async(tw, twg, L);
  k5cg_task<L, XP, LAST, TM>(a, tw, xb, pf, red, wt);   // griddepcontrol.wait inside, after the r prefetch
}

// ------------------------------------------------------------------ row task (one (coil, Omega row) per group)
// Group g of the CTA (T threads) handles pair pair0 + g, pairs ordered coil-major (j * n + yy).
// Groups are independent (each inside one warp); no CTA-wide barrier is used.
template <int L, int MODE>
__device__ __forceinline__ void row_task(const RowArgs& a, int pair0, const float2* tw, float2* xbase,
                                         bool tw_async = false, float2* cst = nullptr) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t H = (size_t)n * L, Q = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;

  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int pair = pair0 + g;
  const bool active = pair < a.J * n;
  const int pc = active ? pair : 0;   // an inactive group (tail of the last CTA) works on row 0 of coil 0
  const int j = pc / n, yy = pc % n, row = q + yy;
  RowBuf buf{xbase + (size_t)g * L};

  if constexpr (MODE == RK_SETPOINT || MODE == RK_SETPOINT_FWD || MODE == RK_RSS) {
    if (active && j == 0)
      for (int i = t; i < n; i += T) a.rho_omega[(size_t)yy * n + i] = a.xrho[(size_t)row * L + q + i];
  }
  float2 v[E];
  // K2 with staging (row_kernel, cst != nullptr): c_j|Omega and rho|Omega of this row do not depend
  // on the previous pass (they are fixed for the Newton step), so they are copied into shared
  // memory BEFORE griddepcontrol.wait and land while the previous pass drains; p_rho (written by
  // the previous pass) follows after the wait. 16-byte cp.async, read back after tw_wait.
  float2* gst = nullptr;
  if constexpr (MODE == RK_K2) {
    if (cst != nullptr) {
      gst = cst + (size_t)g * 3 * n;
      const int jj = active ? j : 0, y2 = active ? yy : 0;
      const float2* srcs[2] = {a.c_omega + jj * Q + (size_t)y2 * n, a.rho_omega + (size_t)y2 * n};
#pragma unroll
      for (int b = 0; b < 2; ++b)
        for (int i = t; i < n / 2; i += T) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(gst + b * n + 2 * i);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(srcs[b] + 2 * i));
        }
      asm volatile("cp.async.commit_group;\n" ::);
      pdl_wait();
      pdl_trigger();
      const float2* pr_src = a.prho + (size_t)(q + y2) * L + q;
      for (int i = t; i < n / 2; i += T) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(gst + 2 * n + 2 * i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(pr_src + 2 * i));
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
  }
  // Unconditional loads: an inactive group (tail of the last CTA) transforms a valid row it never
  // stores. A per-element "if (active)" makes the compiler put each load and its first use in one
  // branch region, which serialises the E load latencies.
  {
    const float2* src = a.in + (size_t)j * H + (size_t)yy * L;
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = src[S::in_idx(t, psh_in<L>(e))];   // half-shifted input (psh_in)
  }
  if (tw_async) tw_wait();
  fft<L, +1>(v, t, tw, buf, SyncWarp{});
  // the centred row IFFT at k = S::out_idx(t, e) is register psh_out(e); only Omega columns are kept
  float2 w[E];
#pragma unroll
  for (int e = 0; e < E; ++e) w[e] = v[psh_out<L>(e)];

  if constexpr (MODE == RK_SETPOINT || MODE == RK_SETPOINT_FWD || MODE == RK_RSS) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = S::out_idx(t, e);
      if (out_is_omega<L>(e)) {
        const float2 cv = w[e];
        if (active) a.c_omega[j * Q + (size_t)yy * n + (k - q)] = cv;
        if constexpr (MODE == RK_SETPOINT_FWD) {
          const float2 rv = active ? a.xrho[(size_t)row * L + k] : make_float2(0.f, 0.f);
          v[e] = cscale(cmul(rv, cv), invL);
        } else if constexpr (MODE == RK_RSS) {
          if (active) a.rss[j * Q + (size_t)yy * n + (k - q)] = cv.x * cv.x + cv.y * cv.y;
        }
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
  } else if constexpr (MODE == RK_K2) {
    float2 cv[E / 2], rv[E / 2], pr[E / 2];
    int u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        if (gst != nullptr) {   // staged rows (valid for inactive groups too: row 0 of coil 0)
          cv[u] = gst[k - q];
          rv[u] = gst[n + (k - q)];
          pr[u] = gst[2 * n + (k - q)];
        } else if (active) {
          cv[u] = a.c_omega[j * Q + (size_t)yy * n + (k - q)];
          rv[u] = a.rho_omega[(size_t)yy * n + (k - q)];
          pr[u] = a.prho[(size_t)row * L + k];
        } else {
          cv[u] = rv[u] = pr[u] = make_float2(0.f, 0.f);
        }
        ++u;
      }
    }
    u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        const float2 dc = w[e];
        const float2 z = cadd(cmul(pr[u], cv[u]), cmul(rv[u], dc));
        v[e] = cscale(z, invL);
        ++u;
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
  } else if constexpr (MODE == RK_K4) {
    float2 cv[E / 2], rv[E / 2];
    int u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        if (active) {
          cv[u] = a.c_omega[j * Q + (size_t)yy * n + (k - q)];
          rv[u] = a.rho_omega[(size_t)yy * n + (k - q)];
        } else {
          cv[u] = rv[u] = make_float2(0.f, 0.f);
        }
        ++u;
      }
    }
    u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        const float2 uu = w[e];
        // per-coil term of sum_j conj(c_j) u_j (Table 1 "sum c_j"); summed in coil order by the consumer
        if (active) a.S[j * Q + (size_t)yy * n + (k - q)] = cmulc(cv[u], uu);
        v[e] = cscale(cmulc(rv[u], uu), invL);
        ++u;
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
  }

  if constexpr (MODE == RK_SETPOINT_FWD || MODE == RK_K2 || MODE == RK_K4) {
    out_to_in<L>(v, t, buf, SyncWarp{});
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_in<L>(e)];   // half-shifted input of the row FFT
    fft<L, -1, omega_shift_zmask<L>()>(w, t, tw, buf, SyncWarp{});   // Omega columns only
    if (active) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        a.out[j * H + (size_t)yy * L + k] = w[psh_out<L>(e)];
      }
    }
  }
}

// K4 as one CTA per Omega row over all local coils (chunks of GPC coils), so the channel sum
// sum_j conj(c_j) u_j (Table 1 "sum c_j") is formed in shared memory in ascending coil order.
template <int L>
__device__ __forceinline__ void row_task_k4(const RowArgs& a, int yy, int jlo, int jhi, int plane, const float2* tw,
                                            float2* xbase, float2* accs, bool tw_async = false, bool pre_wait = false) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C::T, E = C::E;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t H = (size_t)n * L, Q = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int g = tid / T, t = tid % T, GPC = nt / T;

  RowBuf buf{xbase + (size_t)g * L};
  for (int i = tid; i < n; i += nt) accs[i] = make_float2(0.f, 0.f);
  // rho|Omega of this row is shared by every coil
  float2 rv[E / 2];
  {
    int u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (out_is_omega<L>(e)) rv[u++] = __ldcg(a.rho_omega + (size_t)yy * n + (S::out_idx(t, e) - q));
  }
  for (int j0 = jlo; j0 < jhi; j0 += GPC) {
    const int j = j0 + g;
    const bool active = j < jhi;
    float2 v[E], cv[E / 2];
    {  // c_j|Omega is fixed for the Newton step: loaded before griddepcontrol.wait (pre_wait)
      int u = 0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (out_is_omega<L>(e)) {
          // ld.global.cg: L2 is the coherence point for data of an earlier grid read before the wait
          cv[u] = active ? __ldcg(a.c_omega + j * Q + (size_t)yy * n + (S::out_idx(t, e) - q)) : make_float2(0.f, 0.f);
          ++u;
        }
    }
    if (pre_wait && j0 == jlo) {
      pdl_wait();
      pdl_trigger();
    }
    {  // unconditional loads (see row_task); an inactive group's result is masked below
      const float2* src = a.in + (size_t)(active ? j : jlo) * H + (size_t)yy * L;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[S::in_idx(t, psh_in<L>(e))];   // half-shifted (psh_in)
    }
    if (tw_async && j0 == jlo) tw_wait();
    fft<L, +1>(v, t, tw, buf, SyncWarp{});
    float2 w[E];   // centred IFFT at k = out_idx(t, e) (psh_out)
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_out<L>(e)];
    __syncthreads();  // accs / previous chunk's exchange buffers are free
    {
      int u = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (out_is_omega<L>(e)) {
          const int k = S::out_idx(t, e);
          const float2 uu = w[e];
          buf(k - q) = cmulc(cv[u], uu);
          v[e] = cscale(cmulc(rv[u], uu), invL);
          ++u;
        } else {
          v[e] = make_float2(0.f, 0.f);
        }
      }
    }
    __syncthreads();
    for (int xx = tid; xx < n; xx += nt) {
      float2 sacc = accs[xx];
      for (int gg = 0; gg < GPC && j0 + gg < jhi; ++gg) sacc = cadd(sacc, xbase[(size_t)gg * L + xx]);
      accs[xx] = sacc;
    }
    __syncthreads();
    out_to_in<L>(v, t, buf, SyncWarp{});
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_in<L>(e)];
    fft<L, -1, omega_shift_zmask<L>()>(w, t, tw, buf, SyncWarp{});   // Omega columns only
    if (active) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = S::out_idx(t, e);
        a.out[j * H + (size_t)yy * L + k] = w[psh_out<L>(e)];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += nt) a.S[(size_t)plane * Q + (size_t)yy * n + i] = accs[i];
  __syncthreads();
}

// K4 coils per CTA: 64-thread CTAs (whole warps) so the n Omega rows x coil chunks fill the SMs
int k4_chunk_override();  // NLINV_K4CHUNK (0 = default)
int row_pairs_override(); // NLINV_ROWPAIRS (0 = default)
template <int L>
inline int row_pairs_per_cta() {
  const int o = row_pairs_override();
  int g = (o > 0) ? o : 256 / Cfg<L>::T;
  if (g > 256 / Cfg<L>::T) g = 256 / Cfg<L>::T;
  while ((g * Cfg<L>::T) % 32 != 0) ++g;
  return g;
}
template <int L>
inline int k4_chunk_t(int J) {
  const int o = k4_chunk_override();
  int c = (o > 0) ? o : 256 / Cfg<L>::T;
  if (c * Cfg<L>::T > 1024) c = 1024 / Cfg<L>::T;
  return c < J ? c : J;
}

template <int L>
struct RowGeo {
  static constexpr int T = Cfg<L>::T;
  static constexpr int THREADS = 256;
  static constexpr int GPC = THREADS / T;  // (coil, row) pairs per CTA
  static constexpr size_t SMEM = sizeof(float2) * (size_t)L * (GPC + 1) + sizeof(float2) * (L / 2);
  static constexpr size_t SMEM_K2 = sizeof(float2) * ((size_t)L * (GPC + 1) + (size_t)GPC * 3 * (L / 2));
};

// XP: K4 with the peer-memory exchange (its own instantiation). ONE: register bound for one CTA per SM,
// used for K2 when its grid is a single wave of one CTA per SM anyway (C2: 144 CTAs on 148 SMs), where the
// two-CTA bound (128 registers) only makes it spill
// UNST: K2 without the shared-memory staging (grids above one wave whose staging would cost residency);
// the default instantiation of K2 is compiled for the staged path only
template <int L, int MODE, bool XP = false, bool ONE = false, bool UNST = false>
__global__ void __launch_bounds__(256, ONE ? 1 : NLV_MINB) row_kernel(RowArgs a, const float2* __restrict__ twg) {
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  tw_copy_async(tw, twg, L);
  if constexpr (MODE == RK_K4) {
    // CTA = (Omega row, chunk of a.kchunk coils); chunk c writes coil-sum plane c. rho|Omega and
    // c_j|Omega (fixed for the Newton step) are read before griddepcontrol.wait
    const int jlo = blockIdx.y * a.kchunk, jhi = min(a.J, jlo + a.kchunk);
    if constexpr (XP) {
      // peer exchange: the rank's coil-sum plane (one chunk = all local coils) goes straight into
      // the exchange window's buffer of the next epoch; the last CTA publishes it
      RowArgs b = a;
      b.S = xw_S(a.xp->win[a.xp->rank], (int)((x_epoch(*a.xp, XK_S) + 1) & 1ull), (size_t)(L / 2) * (L / 2));
      row_task_k4<L>(b, blockIdx.x, jlo, jhi, 0, tw, xb, xb + (size_t)L * (blockDim.x / Cfg<L>::T), true, true);
      x_publish_last_block(*a.xp, XK_S);
    } else {
      row_task_k4<L>(a, blockIdx.x, jlo, jhi, blockIdx.y, tw, xb, xb + (size_t)L * (blockDim.x / Cfg<L>::T), true, true);
    }
  } else if constexpr (MODE == RK_K2) {
    // per-group staging of c_j|Omega, rho|Omega, p_rho|Omega after the exchange buffers (RowGeo::SMEM_K2)
    const int gpc = blockDim.x / Cfg<L>::T;
    if constexpr (!UNST) {   // the launcher picks the instantiation from its staging decision
      row_task<L, MODE>(a, blockIdx.x * gpc, tw, xb, true, xb + (size_t)L * gpc);
    } else {
      pdl_wait();
      pdl_trigger();
      row_task<L, MODE>(a, blockIdx.x * gpc, tw, xb, true);
    }
  } else {
    pdl_wait();
    pdl_trigger();
    row_task<L, MODE>(a, blockIdx.x * (blockDim.x / Cfg<L>::T), tw, xb, true);
  }
}

// ------------------------------------------------------------------ cluster-fused K2 -> K3 -> K4
// One thread-block cluster per coil runs the three middle passes of the normal operator
// without leaving the chip: CTA b of the C-CTA cluster owns R = 256/T Omega rows
// (the row passes) and W = 2R grid columns (the column pass), and the two row<->column transposes
// go through distributed shared memory (each CTA pulls its operand from the other CTAs' shared
// memory with ld.shared::cluster after a cluster barrier) instead of T2/T3 round trips through L2
// and two kernel boundaries. P:244 (per-channel FFTs + point-wise operations), P:339 (the FFT is the
// most time-consuming operation).
//   phase 1 (K2, rows):    T1 row -> row IFFT -> dc; z = M(p_rho c + rho dc)/L -> row FFT -> X (own, [R][L])
//   cluster barrier; pull my W columns of all n Omega rows from the cluster's X into registers;
//   cluster barrier (every X is free again)
//   phase 2 (K3, columns): column FFT -> x P_k -> column IFFT (Omega rows) -> X (own, [n][W])
//   cluster barrier
//   phase 3 (K4, rows):    pull my R rows (all L columns) from the cluster's X -> row IFFT -> u;
//                          S_j = conj(c_j) u (per-coil plane, summed in coil order by the consumer);
//                          v = conj(rho) u / L -> row FFT -> T4 (global, read by the fused K5 pass)
// Shared memory: twiddles, X (the exchanged data, R*L = n*W values) and D (the FFT exchange buffer),
// ~101 KB at L = 384, i.e. two CTAs per SM so that J clusters of C CTAs are co-resident.
template <int L>
struct K234Geo {
  static constexpr int T = Cfg<L>::T;
  static constexpr int R = 256 / T;          // Omega rows per CTA (row phases: R groups of T threads)
  static constexpr int C = ((L / 2) / R) > 0 ? (L / 2) / R : 1;   // CTAs per cluster (= per coil)
  static constexpr int W = L / C;            // columns per CTA (column phase)
  static constexpr int CW = ColGeo<L>::CW;   // columns per column round
  static constexpr int ROUNDS = W / CW;
  static constexpr bool kOk = (R * T == 256) && (C >= 2) && (C <= 16) && ((L / 2) % R == 0) && (L % C == 0) &&
                              (W % CW == 0) && (ROUNDS == 2) && (CW * T == 256) && (Sched<L>::kSymmetric);
  static constexpr size_t XN = (size_t)R * L;               // == (L/2) * W
  static constexpr size_t SMEM = sizeof(float2) * ((size_t)L + 2 * XN);
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
// shared::cta address of this CTA's buffer -> shared::cluster address of the same buffer in CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ float2 ld_dsmem(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}

template <int L>
__global__ void __launch_bounds__(256, 2) k234_kernel(RowArgs a, const float2* __restrict__ twg) {
  using G = K234Geo<L>;
  using C_ = Cfg<L>;
  using S = Sched<L>;
  constexpr int T = C_::T, E = C_::E, R = G::R, W = G::W, CW = G::CW;
  constexpr int n = L / 2, q = L / 4;
  constexpr size_t H = (size_t)n * L, Q = (size_t)n * n;
  constexpr float invL = 1.0f / (float)L;
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* X = tw + L;          // exchanged data: phase 1 out [R][L], phase 2 out [n][W]
  float2* D = X + G::XN;       // FFT exchange buffer
  const int b = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  tw_copy_async(tw, twg, L);

  // ---- operands fixed for the Newton step / the frame: read before griddepcontrol.wait
  // phase-2 mask bits of this thread's two columns (k-space rows out_idx(t, e))
  const int cc = tid % CW, ct = tid / CW;
  uint32_t mb[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int x = W * b + CW * h + cc;
    uint32_t m = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) m |= (__ldcg(a.mask + (size_t)S::out_idx(ct, e) * L + x) ? 1u : 0u) << e;
    mb[h] = m;
  }
  const int g = tid / T, t = tid % T;
  const int yy = R * b + g;      // Omega row of this group (phases 1 and 3)
  pdl_wait();
  pdl_trigger();

  // ================= phase 1: K2 on row yy
  {
    RowBuf buf{D + (size_t)g * L};
    float2 v[E];
    const float2* src = a.in + (size_t)j * H + (size_t)yy * L;
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = src[S::in_idx(t, psh_in<L>(e))];
    tw_wait();
    fft<L, +1>(v, t, tw, buf, SyncWarp{});
    float2 w[E];
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_out<L>(e)];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        const float2 cv = __ldcg(a.c_omega + (size_t)j * Q + (size_t)yy * n + (k - q));
        const float2 rv = __ldcg(a.rho_omega + (size_t)yy * n + (k - q));
        const float2 pr = a.prho[(size_t)(q + yy) * L + k];
        v[e] = cscale(cadd(cmul(pr, cv), cmul(rv, w[e])), invL);
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_in<L>(e)];
    fft<L, -1, omega_shift_zmask<L>()>(w, t, tw, buf, SyncWarp{});
    float2* xo = X + (size_t)g * L;
#pragma unroll
    for (int e = 0; e < E; ++e) xo[S::out_idx(t, e)] = w[psh_out<L>(e)];
  }
  cluster_sync_all();   // X of every CTA holds its R rows of the row-FFT'd z

  // ================= pull: my W columns of all n Omega rows (column-FFT input pattern, both rounds)
  float2 in2[2][E / 2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int x = W * b + CW * h + cc;
    int u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (in_is_omega<L>(e)) {
        const int yr = S::in_idx(ct, e), r = yr - q;
        const uint32_t ad = dsmem_addr(X + (size_t)(r % R) * L + x, (uint32_t)(r / R));
        in2[h][u++] = cneg_if(ld_dsmem(ad), yr & 1);
      }
    }
  }
  cluster_sync_all();   // every CTA has its inputs: X is free
  // round 1's inputs stay in registers; round 2's are parked in X at their own (row, column) slot of
  // the [n][W] layout, the slot round 2 later overwrites with its output (after the transform's
  // block barriers, i.e. after every parked value has been read back)
  {
    int u = 0;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (in_is_omega<L>(e)) X[(size_t)(S::in_idx(ct, e) - q) * W + CW + cc] = in2[1][u++];
  }

  // ================= phase 2: K3 on columns W b + CW h + cc, two rounds
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    ColBuf<CW> buf{D, cc};
    float2 v[E];
    {
      int u = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (in_is_omega<L>(e)) {
          v[e] = (h == 0) ? in2[0][u] : X[(size_t)(S::in_idx(ct, e) - q) * W + CW + cc];
          ++u;
        } else {
          v[e] = make_float2(0.f, 0.f);
        }
      }
    }
    fft<L, -1, omega_in_zmask<L>()>(v, ct, tw, buf, SyncBlock{});
    const uint32_t mh = (h == 0) ? mb[0] : mb[1];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = ((mh >> e) & 1u) ? v[e] : make_float2(0.f, 0.f);   // (-1)^k signs cancel
    fft<L, +1>(v, ct, tw, buf, SyncBlock{});
    const int xl = CW * h + cc;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(ct, e);
        X[(size_t)(k - q) * W + xl] = cscale(v[e], invL * sgn_of(k));
      }
    }
  }
  cluster_sync_all();   // X of every CTA holds its W columns of the Omega rows

  // ================= phase 3: K4 on row yy
  {
    RowBuf buf{D + (size_t)g * L};
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = S::in_idx(t, psh_in<L>(e));
      v[e] = ld_dsmem(dsmem_addr(X + (size_t)yy * W + (x % W), (uint32_t)(x / W)));
    }
    cluster_arrive();    // this CTA's remote reads are done (waited for before exit)
    fft<L, +1>(v, t, tw, buf, SyncWarp{});
    float2 w[E];
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_out<L>(e)];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (out_is_omega<L>(e)) {
        const int k = S::out_idx(t, e);
        const float2 cv = __ldcg(a.c_omega + (size_t)j * Q + (size_t)yy * n + (k - q));
        const float2 rv = __ldcg(a.rho_omega + (size_t)yy * n + (k - q));
        const float2 uu = w[e];
        a.S[(size_t)j * Q + (size_t)yy * n + (k - q)] = cmulc(cv, uu);   // Table 1 "sum c_j" term of coil j
        v[e] = cscale(cmulc(rv, uu), invL);
      } else {
        v[e] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = v[psh_in<L>(e)];
    fft<L, -1, omega_shift_zmask<L>()>(w, t, tw, buf, SyncWarp{});
    float2* dst = a.out + (size_t)j * H + (size_t)yy * L;
#pragma unroll
    for (int e = 0; e < E; ++e) dst[S::out_idx(t, e)] = w[psh_out<L>(e)];
  }
  cluster_wait();        // no CTA leaves while another may still read its X
}

// ------------------------------------------------------------------ dispatch
template <typename... KArgs, typename... Act>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

template <typename... KArgs, typename... Act>
static cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                               Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  // cooperative (grid barriers); optionally with programmatic dependent launch, so the pass is
  // scheduled while the previous one drains (its CTAs reach a grid barrier only after
  // griddepcontrol.wait, i.e. after the previous pass has released every SM)
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

// CTAs per resident wave of a column kernel, when its grid (L/CW x batch) spans more than one wave and its
// data exceed L2 (next-wave L2 prefetch); 0 otherwise
template <int L, class K>
static int col_wave(K kern, size_t smem, int batch) {
  int dev = 0, nsm = 0, per = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, ColGeo<L>::THREADS, smem) != cudaSuccess || per < 1) return 0;
  const long long wave = (long long)per * nsm, grid = (long long)(L / ColGeo<L>::CW) * batch;
  const double bytes = 8.0 * L * L * batch;
  return (grid > wave && bytes > 0.5 * l2) ? (int)wave : 0;
}

// can the fused K5 + CG + K1 pass (k5cg_kernel) run as one co-resident (cooperative) wave?
template <int L>
static bool k5cg_fusable_l(int J) {
  if (ColGeo<L>::THREADS < 64) return false;
  auto kern = k5cg_kernel<L, false>;
  const size_t smem = ColGeo<L>::SMEM_PF;
  if (cudaFuncSetAttribute(k5cg_kernel<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k5cg_kernel<L, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return false;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, ColGeo<L>::THREADS, smem) != cudaSuccess) return false;
  return (long long)(L / ColGeo<L>::CW) * J <= (long long)per * nsm;
}

template <int L>
static cudaError_t launch_k5cg_t(const ColArgs& a, const float2* tw, cudaStream_t s) {
  auto kern = a.tmap_p != nullptr
                  ? (a.xp != nullptr ? (a.last_iter ? k5cg_kernel<L, true, true> : k5cg_kernel<L, true, false>)
                                     : (a.last_iter ? k5cg_kernel<L, false, true> : k5cg_kernel<L, false, false>))
                  : (a.xp != nullptr ? (a.last_iter ? k5cg_kernel<L, true, true, false> : k5cg_kernel<L, true, false, false>)
                                     : (a.last_iter ? k5cg_kernel<L, false, true, false> : k5cg_kernel<L, false, false, false>));
  const size_t smem = ColGeo<L>::SMEM_PF;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_coop(kern, dim3(L / ColGeo<L>::CW, a.k5_rows > a.J ? a.k5_rows : a.J), dim3(ColGeo<L>::THREADS), smem,
                     s, true, a, tw);
}
// CTA rows of the fused pass: J coil rows; when the coil CTAs alone would leave more than 8 rho elements
// per thread (few local coils: a coil-sharded rank), topped up with rho-only rows to 2 per thread (N / 512
// CTAs), within one co-resident wave. Measured at 384^2 (frames/s, J = 1 / 2 / 4 / 12): 347 / 352 / 346 / 262
// against 249 / 316 / 346 / 263 without rho-only rows; topping up J = 4 (6 per thread) measured slower.
template <int L>
static int k5cg_rows_l(int J) {
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k5cg_kernel<L, false>, ColGeo<L>::THREADS,
                                                    ColGeo<L>::SMEM_PF) != cudaSuccess)
    return J;
  constexpr int NT = L / ColGeo<L>::CW;
  constexpr long long N = (long long)L * L, TH = ColGeo<L>::THREADS;
  if (N <= 8 * TH * NT * (long long)J) return J;
  const long long want = (N + 2 * TH - 1) / (2 * TH);
  long long rows = (want + NT - 1) / NT;
  const long long cap = (long long)per * nsm / NT;
  if (rows > cap) rows = cap;
  return rows > J ? (int)rows : J;
}

template <int L, int MODE>
static cudaError_t launch_col_t(const ColArgs& a, const float2* tw, cudaStream_t s) {
  constexpr bool kPWable = (MODE == CK_PSF || MODE == CK_RESADJ || MODE == CK_FWDP || MODE == CK_ADJ1);
  constexpr bool kXPable = (MODE == CK_FFT_W_NORMAL || MODE == CK_FFT_W_RHS || MODE == CK_FFT_W_ADJ);
  constexpr bool kCG = (MODE == CK_IFFT_W_CG || MODE == CK_FFT_W_NORMAL);
  auto kern = (kPWable && a.pw != nullptr) ? col_kernel<L, MODE, kPWable>
              : (kXPable && a.xp != nullptr) ? col_kernel<L, MODE, false, kXPable>
                                           : col_kernel<L, MODE, false>;
  if constexpr (kCG) {
    if (a.cg1) kern = (kXPable && a.xp != nullptr) ? col_kernel<L, MODE, false, kXPable, true> : col_kernel<L, MODE, false, false, true>;
  }
  if constexpr (MODE == CK_FFT_W_RHS) {
    if (a.fuse_k1) kern = a.xp != nullptr ? col_kernel<L, MODE, false, true, false, true> : col_kernel<L, MODE, false, false, false, true>;
  }
  const size_t smem = ColGeo<L>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(L / ColGeo<L>::CW, a.J);
  return launch_k(kern, grid, dim3(ColGeo<L>::THREADS), smem, s, a, tw);
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
    case CK_K5CG: return launch_k5cg_t<L>(a, tw, s);
  }
  return cudaErrorInvalidValue;
}

template <int L, int MODE>
static cudaError_t launch_row_t(const RowArgs& a0, const float2* tw, cudaStream_t s) {
  const size_t smem = RowGeo<L>::SMEM;
  auto kern = (MODE == RK_K4 && a0.xp != nullptr) ? row_kernel<L, MODE, MODE == RK_K4> : row_kernel<L, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr (MODE == RK_K4) {
    RowArgs a = a0;
    a.kchunk = k4_chunk_t<L>(a.J);
    const size_t sm4 = sizeof(float2) * ((size_t)L * (a.kchunk + 1) + L / 2);
    if (sm4 > smem && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4)) != cudaSuccess)
      return e;
    return launch_k(kern, dim3(L / 2, (a.J + a.kchunk - 1) / a.kchunk), dim3(a.kchunk * Cfg<L>::T), sm4, s, a, tw);
  } else {
    const int gpc = row_pairs_per_cta<L>();
    const int grid = (a0.J * (L / 2) + gpc - 1) / gpc;
    if constexpr (MODE == RK_K2) {
      // staging the pre-wait operands costs shared memory: only where the grid is one wave anyway or two
      // staged CTAs still fit an SM (above L2, e.g. 1024^2 x 32, it would cap the pass at one CTA per SM)
      static int nsm = 0;
      if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      }
      const size_t sm2 = sizeof(float2) * ((size_t)L * (gpc + 1) + (size_t)gpc * 3 * (L / 2));
      RowArgs a = a0;
      a.stage = (sm2 <= 115712 || grid <= nsm) ? 1 : 0;
      const size_t shm = a.stage ? (sm2 > smem ? sm2 : smem) : smem;
      auto k2 = !a.stage ? row_kernel<L, MODE, false, false, true>
                : (grid <= nsm && k2_one_enabled()) ? row_kernel<L, MODE, false, true> : kern;
      if ((e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(shm > smem ? shm : smem))) != cudaSuccess)
        return e;
      return launch_k(k2, dim3(grid), dim3(gpc * Cfg<L>::T), shm, s, a, tw);
    }
    return launch_k(kern, dim3(grid), dim3(gpc * Cfg<L>::T), smem, s, a0, tw);
  }
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

template <int L>
static bool k234_ok_l() {
  if constexpr (!K234Geo<L>::kOk) {
    return false;
  } else {
    auto kern = k234_kernel<L>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K234Geo<L>::SMEM) != cudaSuccess)
      return false;
    if (K234Geo<L>::C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return false;
    return true;
  }
}

template <int L>
static int k234_max_clusters_l() {
  if constexpr (!K234Geo<L>::kOk) {
    return -1;
  } else {
    using G = K234Geo<L>;
    auto kern = k234_kernel<L>;
    if (!k234_ok_l<L>()) return -2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G::C, 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = G::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = G::C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return -3;
    return n;
  }
}

template <int L>
static cudaError_t launch_k234_l(const RowArgs& a, const float2* tw, cudaStream_t s) {
  if constexpr (!K234Geo<L>::kOk) {
    return cudaErrorInvalidConfiguration;
  } else {
    using G = K234Geo<L>;
    auto kern = k234_kernel<L>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return e;
    if (G::C > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G::C, a.J);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = G::C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, a, tw);
  }
}

// Force-load every kernel of this grid size (CUDA lazy loading loads a function at its first launch,
// which can wait for the device to drain: with the peer-memory exchange a rank's kernel may spin on
// a peer whose kernels the host has not enqueued yet, so nothing may be loaded lazily after that)
template <int L>
static cudaError_t preload_l() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  auto get = [&](const void* f) { if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f); };
  get((const void*)col_kernel<L, CK_IFFT_W, false>);
  get((const void*)col_kernel<L, CK_IFFT_W_CG, false>);
  get((const void*)col_kernel<L, CK_FWDP, false>);
  get((const void*)col_kernel<L, CK_FWDP, true>);
  get((const void*)col_kernel<L, CK_PSF, false>);
  get((const void*)col_kernel<L, CK_PSF, true>);
  get((const void*)col_kernel<L, CK_RESADJ, false>);
  get((const void*)col_kernel<L, CK_RESADJ, true>);
  get((const void*)col_kernel<L, CK_ADJ1, false>);
  get((const void*)col_kernel<L, CK_ADJ1, true>);
  get((const void*)col_kernel<L, CK_FFT_W_NORMAL, false>);
  get((const void*)col_kernel<L, CK_FFT_W_RHS, false>);
  get((const void*)col_kernel<L, CK_FFT_W_ADJ, false>);
  get((const void*)k5cg_kernel<L, false>);
  get((const void*)k5cg_kernel<L, true>);
  get((const void*)k5cg_kernel<L, false, true>);
  get((const void*)k5cg_kernel<L, true, true>);
  get((const void*)k5cg_kernel<L, false, false, false>);
  get((const void*)k5cg_kernel<L, true, false, false>);
  get((const void*)k5cg_kernel<L, false, true, false>);
  get((const void*)k5cg_kernel<L, true, true, false>);
  get((const void*)col_kernel<L, CK_FFT_W_NORMAL, false, true>);
  get((const void*)col_kernel<L, CK_FFT_W_RHS, false, true>);
  get((const void*)col_kernel<L, CK_FFT_W_ADJ, false, true>);
  get((const void*)col_kernel<L, CK_IFFT_W_CG, false, false, true>);
  get((const void*)col_kernel<L, CK_FFT_W_NORMAL, false, false, true>);
  get((const void*)col_kernel<L, CK_FFT_W_NORMAL, false, true, true>);
  get((const void*)col_kernel<L, CK_FFT_W_RHS, false, false, false, true>);
  get((const void*)col_kernel<L, CK_FFT_W_RHS, false, true, false, true>);
  get((const void*)row_kernel<L, RK_K4, true>);
  get((const void*)row_kernel<L, RK_SETPOINT>);
  get((const void*)row_kernel<L, RK_SETPOINT_FWD>);
  get((const void*)row_kernel<L, RK_RSS>);
  get((const void*)row_kernel<L, RK_K2>);
  get((const void*)row_kernel<L, RK_K2, false, true>);
  get((const void*)row_kernel<L, RK_K2, false, false, true>);
  get((const void*)row_kernel<L, RK_K4>);
  if constexpr (K234Geo<L>::kOk) get((const void*)k234_kernel<L>);
  return e;
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
  for (int e = 0; e < E; ++e) v[e] = cneg_if(in[(active ? rowi * L : 0) + S::in_idx(t, e)], S::in_idx(t, e) & 1);
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
__global__ void __launch_bounds__(ColGeo<L>::THREADS) fft_cols_tw_kernel(float2* data, const float2* __restrict__ twg,
                                                                         int wave) {
  using C = Cfg<L>;
  using S = Sched<L>;
  constexpr int E = C::E, CW = ColGeo<L>::CW;
  constexpr size_t N = (size_t)L * L;
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* xb = tw + L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
  __syncthreads();
  const int tid = threadIdx.x, c = tid % CW, t = tid / CW;
  const int x = blockIdx.x * CW + c;
  float2* d = data + (size_t)blockIdx.y * N;
  prefetch_next_wave_cols<L>(data, N, wave, 0, L);
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
    ck<<<dim3(L / ColGeo<L>::CW, batch), ColGeo<L>::THREADS, csm, s>>>(out, tw, col_wave<L>(ck, csm, batch));
  } else {
    auto rk = fft_rows_tw_kernel<L, -1>;
    auto ck = fft_cols_tw_kernel<L, -1>;
    if ((e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm)) != cudaSuccess) return e;
    rk<<<(nrows + gpc - 1) / gpc, gpc * T, rsm, s>>>(in, out, nrows, tw);
    ck<<<dim3(L / ColGeo<L>::CW, batch), ColGeo<L>::THREADS, csm, s>>>(out, tw, col_wave<L>(ck, csm, batch));
  }
  return cudaGetLastError();
}

// Per-grid-size entry points, defined in one translation unit per size (inst.cu -DNLV_L=...).
#define NLV_DECLARE(L)                                                                           \
  cudaError_t launch_col_##L(int mode, const ColArgs& a, const float2* tw, cudaStream_t s);     \
  cudaError_t launch_row_##L(int mode, const RowArgs& a, const float2* tw, cudaStream_t s);     \
  cudaError_t launch_fft2d_##L(const float2* in, float2* out, int batch, int inverse, const float2* tw, \
                               cudaStream_t s);                                                 \
  int col_tiles_##L();                                                                          \
  bool k5cg_fusable_##L(int J);                                                                  \
  int k5cg_rows_##L(int J);                                                                      \
  bool k234_ok_##L();                                                                            \
  cudaError_t launch_k234_##L(const RowArgs& a, const float2* tw, cudaStream_t s);              \
  int k234_max_clusters_##L();                                                                   \
  cudaError_t preload_##L();
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
  int col_tiles_##L() { return L / ColGeo<L>::CW; }                                             \
  bool k5cg_fusable_##L(int J) { return k5cg_fusable_l<L>(J); }                                  \
  int k5cg_rows_##L(int J) { return k5cg_rows_l<L>(J); }                                          \
  bool k234_ok_##L() { return k234_ok_l<L>(); }                                                  \
  cudaError_t launch_k234_##L(const RowArgs& a, const float2* tw, cudaStream_t s) { return launch_k234_l<L>(a, tw, s); } \
  int k234_max_clusters_##L() { return k234_max_clusters_l<L>(); }                                 \
  cudaError_t preload_##L() { return preload_l<L>(); }

#define NLV_FOR_EACH_NG(X) X(16) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384) X(512) X(768) X(1024)
NLV_FOR_EACH_NG(NLV_DECLARE)

}  // namespace nlv
