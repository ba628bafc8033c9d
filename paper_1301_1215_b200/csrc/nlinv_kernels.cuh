// Internal interface between the C-ABI host code (nlinv_capi.cu) and the sm_100a kernels
// (nlinv_kernels.cu). Not part of the public boundary (include/nlinv.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nlv {

// Scalar slots (doubles) written once per CG solve and read by later kernels.
constexpr int kMaxCG = 512;
constexpr int kMaxNewton = 64;
constexpr int SC_RR_RHO = 0;                         // <r_i, r_i> rho block     [kMaxCG + 1]
constexpr int SC_RR_CHAT = SC_RR_RHO + kMaxCG + 1;   // <r_i, r_i> chat blocks   [kMaxCG + 1]
constexpr int SC_PAP_RHO = SC_RR_CHAT + kMaxCG + 1;  // Re<p_i, A p_i> rho       [kMaxCG]
constexpr int SC_PAP_CHAT = SC_PAP_RHO + kMaxCG;     // Re<p_i, A p_i> chat      [kMaxCG]
constexpr int SC_RES = SC_PAP_CHAT + kMaxCG;         // ||P y - F(x_n)||^2       [kMaxNewton]
constexpr int SC_RAP_RHO = SC_RES + kMaxNewton;      // Re<r_i, A p_i> rho  (single-reduction CG, R19)
constexpr int SC_RAP_CHAT = SC_RAP_RHO + kMaxCG;     // Re<r_i, A p_i> chat
constexpr int SC_AA_RHO = SC_RAP_CHAT + kMaxCG;      // <A p_i, A p_i> rho
constexpr int SC_AA_CHAT = SC_AA_RHO + kMaxCG;       // <A p_i, A p_i> chat
constexpr int SC_TOTAL = SC_AA_CHAT + kMaxCG;

// Reduction slots (each has its own partial array and arrival counter).
enum RedSlot { RS_A = 0, RS_B = 1, RS_C = 2, RS_COUNT = 3 };
constexpr int kMaxRedBlocks = 8192;

// Column-kernel modes (one CTA = CW adjacent columns of one coil).
enum ColMode {
  CK_IFFT_W = 0,   // K1 / set-point: t = w^-1 src / ng -> column IFFT -> Omega rows
  CK_IFFT_W_CG,    // K1 with fused CG direction update p = r + beta p (+ rho-block slice)
  CK_FWDP,         // forward / derivative tail: column FFT -> x P -> full k-space
  CK_PSF,          // K3: column FFT -> x P -> column IFFT -> Omega rows
  CK_RESADJ,       // Newton: column FFT -> r = P(y - F x) (+||r||^2) -> column IFFT -> Omega rows
  CK_ADJ1,         // adjoint head: P dy -> column IFFT -> Omega rows
  CK_FFT_W_NORMAL, // K5: column FFT -> Ap = w^-1 . + alpha p (+<p,Ap>)
  CK_FFT_W_RHS,    // Newton rhs: b = w^-1 . - alpha (chat - chat_ref); r = p = b (+<b,b>)
  CK_FFT_W_ADJ,    // adjoint tail: w^-1 . (no alpha)
  CK_K5CG,         // K5 + CG step + K1 (or Newton update), one grid barrier (k5cg_kernel)
};

// Row-kernel modes (one CTA = one Omega row of all local coils).
enum RowMode {
  RK_SETPOINT = 0,  // row IFFT -> c_j on Omega (+ rho|Omega cache)
  RK_SETPOINT_FWD,  // ... and z = rho c_j -> row FFT (forward operator head)
  RK_RSS,           // row IFFT -> c_j, sum_j |c_j|^2 on Omega (frame output)
  RK_K2,            // row IFFT -> dc; z = p_rho c + rho dc -> row FFT
  RK_K4,            // row IFFT -> u; S += conj(c) u; v = conj(rho) u -> row FFT
};

// ------------------------------------------------------------------ peer-memory exchange
// The coil-sharded multi-GPU path's exchanges go through every rank's exchange window, a device
// allocation the other ranks map (CUDA IPC between processes, plain pointers inside one process):
// the modern analogue of the paper's peer-to-peer all-reduce kernel kern_all_red_p2p_2d
// (P:280-289), with loads over NVLink instead of PCIe copies, fused into the kernels that produce
// and consume the data.
//   kind XK_S:    the local coil-sum plane of the Omega window (K4 output), double-buffered by epoch
//   kind XK_DOTS: the fused K5 pass's 8 dot partials (rho, chat parts), double-buffered by epoch
//   kinds XK_A/B: arrive / ack flags of the generic two-phase exchange (xchg_kernel)
// A rank publishes epoch e of kind k by a release store of e into its own flag k after the data of
// e are written; a consumer waits (acquire loads) until every rank's flag k >= e and then reads every
// rank's buffer [e % 2] in ascending rank order. Double buffering is safe because a rank produces
// epoch e only after it consumed e - 1, i.e. after every peer published e - 1, which every peer does
// only after it finished reading e - 2 (stream order).
constexpr int kMaxRanks = 8;
enum XKind { XK_S = 0, XK_DOTS = 1, XK_A = 2, XK_B = 3, XK_COUNT = 4 };
struct XPeers {
  char* win[kMaxRanks];    // every rank's exchange window, [rank] = this rank's own
  int G;                   // ranks (0: exchange off)
  int rank;
};
constexpr size_t kXWinHdr = 4096;   // flags [kind * 128], counters [1024 + kind * 128], dots [2048], xs [2304]
constexpr int kXsSlots = 192;       // generic exchange scalars (doubles)
inline size_t xwin_bytes(size_t Q) { return kXWinHdr + 2 * Q * 8 + Q * 4; }

struct ColArgs {
  const float2* in;        // [J][n][ng] half image (Omega rows) or full k-space input
  float2* out;             // [J][n][ng] half image, or [J][ng][ng] k-space output
  const float2* src;       // chat-type operand [J][ng][ng]
  const float2* src2;      // second operand (chat_ref for RHS, p for NORMAL)
  const float* winv;       // [ng][ng]
  const uint8_t* mask;     // [ng][ng] P_k
  const float* pw;         // [ng][ng] real-valued P_k = sqrt(PSF) of KB gridding (R22); nullptr = binary mask
  const float2* y;         // frame [J][ng][ng]
  float2* r;               // CG residual (chat blocks)
  float2* p;               // CG direction (chat blocks)
  float2* rho_r;           // rho block residual (CG slice of K1)
  float2* rho_p;           // rho block direction
  const double* scal;      // scalar slots
  double* scal_w;
  double* partials;        // reduction partials for this launch
  unsigned* counter;
  int out_slot;            // scalar index the finished reduction is written to (-1: none)
  int out_slot_rho;        // scalar index of the rho-block partial (FFT_W modes)
  float beta;              // CG beta / gamma for CK_IFFT_W_CG (set by the launcher / frame kernel)
  float gamma;
  float2* dx;              // CG solution increment (chat blocks), updated in K1
  float2* rho_dx;
  int nS;                  // number of [n][n] planes of S summed (in order) by the rho slice
  const float2* S;         // coil-sum planes [nS][n][n] (rho slice of the FFT_W modes)
  const float2* rho_a;     // rho-slice operand (p_rho for NORMAL, rho for RHS)
  const float2* rho_b;     // rho_ref for RHS
  float2* rho_out;         // rho-slice output (Ap_rho / adjoint rho)
  unsigned long long* trace;  // debug timeline (-DNLV_TRACE builds only)
  int last_iter;           // k5cg: last CG iteration (Newton update instead of the next K1)
  unsigned* bar_count;     // k5cg: grid barrier word
  double* fpart;           // k5cg: [8 * blocks] dot partials
  int fuse_k1;             // k5cg / rhs: also run K1 of the next CG iteration (T1 into t1)
  float2* t1;              // K1 output (half image) for the fused passes
  float2* xc;              // unknowns, chat blocks (fused Newton update)
  float2* x_rho;           // unknowns, rho block
  int iter;                // CG iteration (beta for CK_IFFT_W_CG)
  int cg1;                 // unfused single-reduction CG (R19): K5 also forms <r,Ap>, <Ap,Ap>, <r,r>;
                           // K1 applies r -= gamma Ap (A p from src2 / rho_a) before the p update
  float alpha;
  int J;
  const XPeers* xp;        // peer-memory exchange (world > 1 without NCCL): device copy; nullptr: off
  const void* tmap_r;      // k5cg: CUtensorMap (device, 64-B aligned) of the chat blocks of r / dx for the TMA
  const void* tmap_dx;     // tile prefetch; nullptr: cp.async prefetch
  int k5_rows;              // k5cg: CTA rows (>= J; rows >= J are rho-only CTAs)
  int fold_sp;              // k5cg, last CG iteration: also the set-point column pass of x_{n+1} into t1
  const void* tmap_p;      // k5cg: CUtensorMap of the chat blocks of p: the p tile lands in the FFT exchange buffer
                           // (where p is parked) right after the column FFT's last exchange; nullptr: global loads
};

struct RowArgs {
  const float2* in;        // [J][n][ng]
  float2* out;             // [J][n][ng]
  float2* c_omega;         // [J][n][n]
  float2* rho_omega;       // [n][n]
  const float2* xrho;      // rho of the point, full grid (set point)
  const float2* prho;      // rho part of the direction, full grid (K2)
  float2* S;               // K4: coil-sum planes [chunks][n][n] (ordered within a chunk)
  float* rss;              // [J][n][n] per-coil |c_j|^2 (RSS)
  const uint8_t* mask;     // [ng][ng] P_k (cluster-fused K2-K3-K4)
  int J;
  const XPeers* xp;        // peer-memory exchange: K4 writes its coil-sum plane into the window and publishes
  int kchunk;              // K4 coils per CTA (set by the launcher)
  int stage;               // K2: stage c|Omega, rho|Omega, p_rho rows in shared memory (set by the launcher)
};
int k4_planes(int ng, int J);  // number of K4 coil-sum planes
int fft_radices(int ng, int* R);  // radices R[0..NP-1] of the length-ng transform's Stockham passes; returns NP

struct VecArgs {
  float2* x;         // unknowns (CG update of the last iteration adds into x)
  float2* dx;
  float2* r;
  float2* p;
  const float2* Ap;
  const float2* S;       // all-reduced coil sum [n][n]
  const float2* xref;
  float2* out;
  const double* scal;
  double* scal_w;
  double* partials;
  unsigned* counter;
  int iter;
  int last;
  float alpha;
  long long nrho;        // elements in the rho block (N)
  long long ntot;        // elements in all blocks ((1+J) N)
};

// launchers (return cudaGetLastError())
cudaError_t launch_col(int ng, int mode, const ColArgs& a, const float2* tw, cudaStream_t s);
cudaError_t launch_row(int ng, int mode, const RowArgs& a, const float2* tw, cudaStream_t s);
cudaError_t launch_newton_update(int ng, const VecArgs& a, cudaStream_t s);
cudaError_t launch_r_update(int ng, const VecArgs& a, cudaStream_t s);
cudaError_t launch_image(int ng, const float2* rho_omega, const float* rss, int nplanes, float2* img, cudaStream_t s);
cudaError_t launch_fft2d(int ng, const float2* in, float2* out, int batch, int inverse, const float2* tw,
                         float2* tmp, cudaStream_t s);
bool supported_ng(int ng);
bool pdl_enabled();
bool k2_one_enabled();
int col_tiles(int ng);  // column-kernel CTAs per coil
cudaError_t launch_init_x(float2* x, long long nrho, long long ntot, cudaStream_t s);
cudaError_t launch_mask_compact(const uint8_t* mask, int N, int* counts, int* idx, int* nnz, cudaStream_t s);
int mask_count_blocks(int N);
cudaError_t launch_grid_radial(const float2* raw, int J, int nraw, const int* cells, const int* start, const int* sid,
                               const float* wgt, int nnz, size_t N, float2* y, cudaStream_t s);
cudaError_t launch_scatter_samples(const float2* samples, const int* idx, const int* nnz, int nnz_cap, int J,
                                   size_t N, float2* y, cudaStream_t s);
bool k5cg_fusable(int ng, int J);
int k5cg_rows(int ng, int J);   // CTA rows of the fused pass (>= J: the extra rows carry rho stripes only)
// cluster-fused K2 -> K3 -> K4 (one thread-block cluster per coil, DSMEM transposes)
bool k234_supported(int ng);
cudaError_t launch_k234(int ng, const RowArgs& a, const float2* tw, cudaStream_t s);
int k234_max_clusters(int ng);
// load every kernel the plan may launch (no lazy loading once peers may spin on each other)
cudaError_t preload_kernels(int ng);
cudaError_t launch_coil_sum(int ng, const float2* S_all, int J, float2* S, cudaStream_t s);
// generic two-phase peer exchange (one CTA): nsum scalars summed over ranks (slots src[i] -> dst[i] of
// scal), nr0 scalars taken from rank 0, and optionally the RSS plane (rss_local [Q] of every rank summed
// into rss_out). Arrive, wait, reduce, ack, wait, then write (so every buffer is reusable afterwards).
struct XchgArgs {
  XPeers xp;
  double* scal;
  int nsum, nr0;
  int src[64], dst[64];    // first nsum: summed; next nr0: rank 0's value
  float* rss_out;          // nullptr: no RSS plane
  int Q;
};
cudaError_t launch_xchg(const XchgArgs& a, cudaStream_t s);
cudaError_t launch_axpy(float a, const float* x, float* y, long long n, cudaStream_t s);
cudaError_t launch_rss_sum(int ng, const float* rss_all, int J, float* rss, cudaStream_t s);

}  // namespace nlv
