/*
 * nlinv.h -- C ABI of the B200 NLINV / IRGNM hot path (libnlinv.so).
 *
 * The method (Schaetz & Uecker, arXiv:1301.1215, "PAPER.md"):
 *   unknowns x = (rho, chat_1..chat_J): image and weighted-domain coil sensitivities,
 *                jointly estimated
 *   F  = P_k DTFT M_Omega C W^{-1}                                         (Eq. 2)
 *   IRGNM step: (DF^H DF + alpha_n I)(x_{n+1} - x_n)
 *                 = DF^H (y - F x_n) - alpha_n (x_n - x_ref),  solved by CG (Eq. 3)
 *   multi-GPU:  coils are distributed over the GPUs, rho = sum_g rho_g is a block-wise
 *               all-reduce after every channel summation
 *
 * Conventions shared by every call (readings R1-R13 in DESIGN.md):
 *   - Grid: square ng x ng (nx == ny == ng), ng in {16,32,48,64,96,128,192,256,384,512,768,1024}
 *     (the paper's matrix 192-384 doubled to 384-768). n = ng/2.
 *     Omega = centred n x n square: rows/cols ng/4 .. 3ng/4-1 (R3).
 *   - Complex single precision, interleaved (re, im) == nlinv_c32 == torch.complex64,
 *     row-major [.., y, x], x fastest. Centred unitary 2D DFT (R1).
 *   - Unknown-vector layout on a rank that owns coils [first, first+count):
 *         [ rho (ng*ng) | chat_first .. chat_{first+count-1} (count*ng*ng) ]
 *     rho is replicated on every rank ("all GPUs require rho").
 *   - k-space arrays (frame y, operator outputs): [count][ng][ng], local coils only.
 *   - Device pointers are caller-owned, must live on the plan's device, be 16-byte aligned,
 *     and are borrowed only for the duration of the (stream-ordered) call. Every device call
 *     enqueues on `stream` (a cudaStream_t, NULL = legacy default stream) and returns without
 *     a host synchronisation. Buffers passed to one call must not overlap unless stated.
 *   - Synchronous argument errors (NLINV_ERR_ARG / _SIZE / _STATE) are returned before anything
 *     is enqueued. CUDA / NCCL launch errors are returned as NLINV_ERR_CUDA / _NCCL and latched
 *     (nlinv_last_error). Numerical events (CG breakdown, divergence) are flags read by
 *     nlinv_plan_stats, not errors.
 *   - Not thread-safe per plan; one plan per rank/device. No exceptions cross this ABI.
 */
#ifndef NLINV_H_
#define NLINV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nlinv_plan_s* nlinv_plan;
typedef struct { float re, im; } nlinv_c32;

typedef enum {
  NLINV_OK = 0,
  NLINV_ERR_ARG = 1,       /* null pointer / bad scalar argument */
  NLINV_ERR_SIZE = 2,      /* unsupported grid, coil count or iteration count */
  NLINV_ERR_STATE = 3,     /* e.g. derivative before set_point */
  NLINV_ERR_CUDA = 4,
  NLINV_ERR_NCCL = 5,
  NLINV_ERR_NOMEM = 6,
  NLINV_ERR_DIVERGED = 7,  /* reported by nlinv_plan_stats only */
  NLINV_ERR_NOT_BUILT = 8  /* library built without NCCL and world > 1 */
} nlinv_status;

typedef struct {
  float sob_a, sob_b;   /* W: w(k) = (1 + a|k|^2)^(b/2), k in [-1/2,1/2)^2; default 220, 32 (R2) */
  float alpha0, q;      /* alpha_n = alpha0 q^n, restarted each frame; default 1, 1/3 (R4) */
  int fov_full;         /* must be 0: Omega = centred n x n (the whole-grid variant exists only in the
                           oracle's closed-form pins; ERR_ARG here) */
  int rank, world;      /* coil shard of this process; default 0, 1 */
  const unsigned char* nccl_id;  /* world > 1: 128-byte ncclUniqueId from nlinv_get_unique_id (rank 0) for
                                    the NCCL transport, or NULL for the peer-memory exchange
                                    (nlinv_plan_connect*, the default of bench.py) */
} nlinv_params;

typedef struct {
  int newton_done;          /* Newton steps run by the last nlinv_reconstruct */
  int cg_breakdown;         /* 1 if some CG solve hit <r,r> == 0 exactly (all later steps 0; A9) */
  int diverged;             /* 1 if ||P y - F x_n|| grew > 10x over its first value */
  double residual[64];      /* ||P y - F(x_n)||_2 per Newton step (Table 1, row F, column A.B; R8) */
} nlinv_stats;

/* Fill *p with the defaults above. */
void nlinv_params_default(nlinv_params* p);

/* Human-readable name of a status. Never NULL. */
const char* nlinv_status_string(nlinv_status s);

/* Last latched error message of a plan (or of the library when plan == NULL). Never NULL. */
const char* nlinv_last_error(nlinv_plan plan);

/* Library build info: "sm_100a nccl=<0|1> ...". Never NULL. */
const char* nlinv_build_info(void);

/* Rank 0 creates the 128-byte NCCL unique id that every rank passes in nlinv_params.nccl_id.
 * id: host buffer of 128 bytes. ERR_NOT_BUILT without NCCL. */
nlinv_status nlinv_get_unique_id(unsigned char id[128]);

/* Radial sampling pattern P_k (P:346 radial; P:233 gridding onto the Cartesian grid), rule R12:
 * spoke s of frame f at theta = pi (s*turns + f mod turns) / (spokes*turns), ng samples at
 * r = i - ng/2, cell (ng/2 + round(r sin theta), ng/2 + round(r cos theta)) with v snapped to the
 * 2^-20 grid and rounded half away from zero; duplicates OR, out-of-grid samples dropped.
 * out: host uint8 [ny][nx], written with 0/1. Host-only, integer-exact. ERR_SIZE if nx != ny,
 * ERR_ARG on bad counts, ERR_STATE if a sample falls within 1e-6 of a snap midpoint. */
nlinv_status nlinv_radial_mask(int nx, int ny, int spokes, int turns, int frame, uint8_t* out);

/* Create a plan on the CURRENT CUDA device.
 * nx, ny: grid (must be equal, see conventions). ncoils: total coils J over all ranks (1..256).
 * mask: host uint8 [ny][nx] sampling pattern P_k (nonzero = sampled); copied.
 * p: NULL = defaults. With world > 1 and p->nccl_id the plan creates its own NCCL communicator
 *    (collective: every rank must call) and runs the unfused CG passes with NCCL all-reduces; with
 *    world > 1 and no nccl_id it runs the fused passes with the peer-memory exchange (connect the
 *    ranks with nlinv_plan_connect* before use). Allocates the whole workspace (no allocation later).
 * out: receives the plan. */
nlinv_status nlinv_plan_create(int nx, int ny, int ncoils, const uint8_t* mask, const nlinv_params* p,
                               nlinv_plan* out);

/* Replace the plan's P_k. mask_host: host uint8 [ng][ng] (synchronous copy, after the plan's last
 * enqueued frame has finished reading the previous P_k).
 * nlinv_plan_set_mask_device: device uint8 [ng][ng], copied on `stream` (per-frame spoke rotation). */
nlinv_status nlinv_plan_set_mask(nlinv_plan plan, const uint8_t* mask_host);
nlinv_status nlinv_plan_set_mask_device(nlinv_plan plan, const uint8_t* mask_dev, void* stream);

/* The coil split rule on its own (host, no device needed): rank `rank` of `world` owns coils
 * [*first, *first + *count): contiguous blocks, the remainder to the low ranks (R10).
 * ERR_ARG unless 1 <= world <= ncoils and 0 <= rank < world. */
nlinv_status nlinv_coil_partition(int ncoils, int world, int rank, int* first, int* count);

/* Coils owned by this rank: contiguous block, remainder to the low ranks (R10). */
nlinv_status nlinv_plan_local_coils(nlinv_plan plan, int* first, int* count);

/* Release everything the plan owns (waits for its work to finish). NULL is a no-op. */
nlinv_status nlinv_plan_destroy(nlinv_plan plan);

/* Linearisation point: c_j = W^{-1} chat_j = F_c^H(w^{-1} chat_j) on Omega, and rho|Omega,
 * are cached in the plan ("F is only required once per Newton step").
 * x: device unknowns (layout above). */
nlinv_status nlinv_set_point(nlinv_plan plan, const nlinv_c32* x, void* stream);

/* y = F(x) = P_k F_c(M_Omega rho c_j) for the local coils (Eq. 2); also sets the point to x.
 * x: device unknowns; y: device [count][ng][ng]. */
nlinv_status nlinv_apply_forward(nlinv_plan plan, const nlinv_c32* x, nlinv_c32* y, void* stream);

/* dy = DF_x dx = P_k F_c(M_Omega (drho c_j + rho W^{-1} dchat_j)) at the cached point (Eq. 3).
 * dx: device unknowns; dy: device [count][ng][ng]. ERR_STATE before any set_point. */
nlinv_status nlinv_apply_derivative(nlinv_plan plan, const nlinv_c32* dx, nlinv_c32* dy, void* stream);

/* dx = DF_x^H dy = ( M sum_j conj(c_j) u_j , { w^{-1} F_c(conj(rho) u_j) }_j ),
 * u_j = M F_c^H(P_k dy_j) at the cached point (Eq. 3; Table 1 row DF^H: the channel sum is
 * all-reduced over ranks). dy: device [count][ng][ng]; dx: device unknowns. */
nlinv_status nlinv_apply_adjoint(nlinv_plan plan, const nlinv_c32* dy, nlinv_c32* dx, void* stream);

/* out = (DF_x^H DF_x + alpha I) dx at the cached point (Eq. 3 left-hand side; the CG operator).
 * dx, out: device unknowns (must not overlap). */
nlinv_status nlinv_apply_normal(nlinv_plan plan, float alpha, const nlinv_c32* dx, nlinv_c32* out,
                                void* stream);

/* One frame of NLINV: newton_steps IRGNM steps (Eq. 3) with alpha_n = alpha0 q^n, each solved
 * by exactly cg_iters textbook CG iterations from 0 (R5, R9).
 * frame:  device [count][ng][ng], the local coils' k-space on the grid; only P_k . frame is
 *         used (samples off P_k are ignored, so a fully gridded or a zero-filled frame both work).
 * prior:  device unknowns used as x_0 = x_ref (the previous frame), or NULL for
 *         x_0 = x_ref = (rho = 1, chat = 0) (R6). May equal x_out.
 * x_out:  device unknowns, receives x_K (the next frame's prior).
 * image_out: device [n][n] complex, crop_Omega(rho . sqrt(sum_j |c_j|^2)) of x_K (R13), or NULL.
 *         With world > 1 every rank receives the full image.
 * Limits: 1 <= cg_iters <= 512, 0 <= newton_steps <= 64.
 * Execution: the frame is captured once into a CUDA graph per (buffers, K, L, P_k kind) and
 * replayed; on the legacy default stream (stream == NULL) the graph runs on a plan-owned stream
 * fenced by events on both sides, so the call stays ordered with `stream`. With a Kaiser-Bessel
 * trajectory active (nlinv_plan_set_trajectory_kb + nlinv_grid_radial) P_k is real-valued (R22). */
nlinv_status nlinv_reconstruct(nlinv_plan plan, const nlinv_c32* frame, const nlinv_c32* prior,
                               int newton_steps, int cg_iters, nlinv_c32* x_out, nlinv_c32* image_out,
                               void* stream);

/* End-to-end variant with HOST buffers: copies frame (host [count][ng][ng]) and optional prior
 * (host unknowns) to the device through the plan's pinned staging, reconstructs, and copies
 * x_out (host unknowns, may be NULL) and image_out (host [n][n], may be NULL) back.
 * Synchronises `stream` before returning. */
nlinv_status nlinv_reconstruct_host(nlinv_plan plan, const nlinv_c32* frame, const nlinv_c32* prior,
                                    int newton_steps, int cg_iters, nlinv_c32* x_out,
                                    nlinv_c32* image_out, void* stream);

/* Real-time streaming entry with HOST buffers (the call a scanner-side user makes per frame).
 * frame_host: [count][ng][ng] k-space of the local coils (pinned memory for full speed).
 * mask_host:  this frame's P_k, host uint8 [ng][ng], or NULL to keep the current one.
 * image_host: [n][n] output (may be NULL).
 * The plan keeps x on the device: the first frame after plan creation / nlinv_stream_reset starts
 * from x_0 = x_ref = (1, 0); every later frame uses the previous frame's x as x_0 = x_ref, the
 * temporal regularisation that makes frames sequential. Synchronises `stream`. */
nlinv_status nlinv_stream_frame(nlinv_plan plan, const nlinv_c32* frame_host, const uint8_t* mask_host,
                                int newton_steps, int cg_iters, nlinv_c32* image_host, void* stream);
nlinv_status nlinv_stream_reset(nlinv_plan plan);

/* The sampled cells of the plan's current P_k as ascending linear indices y*ng + x (
 * integer-exact, computed on the device by stream compaction). idx_host: host int[cap] or NULL
 * (count only); *nnz_host receives the count. ERR_SIZE if cap < count. Synchronises `stream`. */
nlinv_status nlinv_mask_indices(nlinv_plan plan, int* idx_host, int cap, int* nnz_host, void* stream);

/* Streaming entry with a COMPACT frame: samples_host holds, for each local coil, the gridded
 * k-space values at the sampled cells of this frame's P_k in ascending linear-index order
 * ([count][nnz], nnz = number of sampled cells, as nlinv_mask_indices returns). This is the same
 * gridded frame as nlinv_stream_frame without its zeros (after gridding every operation
 * is on the grid; only P_k . y enters the method, R16), ~3.7 % of the bytes at C2. mask_host:
 * this frame's P_k (host uint8 [ng][ng]) or NULL to keep the current one. Synchronises. */
nlinv_status nlinv_stream_frame_compact(nlinv_plan plan, const nlinv_c32* samples_host, int nnz,
                                        const uint8_t* mask_host, int newton_steps, int cg_iters,
                                        nlinv_c32* image_host, void* stream);

/* Per-kernel timing: with profiling on, reconstruct/operator calls run without CUDA graphs and
 * bracket every kernel with CUDA events on its stream. nlinv_plan_profile_json synchronises and
 * writes {"kernel": [launches, total_ms], ...} into buf (ERR_SIZE if len is too small), then
 * clears the record. */
nlinv_status nlinv_plan_set_profiling(nlinv_plan plan, int on);
nlinv_status nlinv_plan_profile_json(nlinv_plan plan, char* buf, size_t len);

/* Debug (builds with -DNLV_TRACE only record data): col_mode >= 0 starts recording per-CTA
 * %globaltimer timelines (8 stamps per CTA) of the column pass with that internal mode;
 * col_mode < 0 copies up to cap stamps into out and stops recording. */
nlinv_status nlinv_plan_trace(nlinv_plan plan, int col_mode, unsigned long long* out, int cap);

/* Statistics of the last reconstruct (synchronises the plan's last stream). */
nlinv_status nlinv_plan_stats(nlinv_plan plan, nlinv_stats* out);

/* Test / micro-benchmark entry: batched centred unitary 2D DFT F_c (inverse = 0) or F_c^H
 * (inverse = 1) of `batch` ng x ng images, the transform every operator is built from.
 * in, out: device [batch][ng][ng]; in == out allowed. */
nlinv_status nlinv_debug_fft2d(nlinv_plan plan, const nlinv_c32* in, nlinv_c32* out, int batch, int inverse,
                               void* stream);

/* ---------------------------------------------------------------------------------------------
 * Peer-memory exchange of the coil-sharded multi-GPU path (PAPER P:246
 * "rho = sum^G rho_g", P:280-289 the peer-to-peer all-reduce kernel, P:339 the exchange inside
 * DF^H, P:370 other decompositions). A plan created with world > 1 and nccl_id == NULL owns an
 * exchange window in device memory; every rank's K4 pass writes its coil-sum plane there and the
 * consumers (the fused K5 + CG pass, the Newton right-hand side) read all ranks' planes over
 * NVLink in ascending rank order, with the CG dot products exchanged the same way inside the fused
 * pass (no NCCL call inside a frame; rho replicas stay bit-identical: the replicated rho parts of
 * the dots are taken from rank 0). Before the first operator call every rank connects to all
 * ranks' windows (ERR_STATE otherwise):
 *   nlinv_plan_exchange_handle: the 64-byte cudaIpcMemHandle_t of this plan's window (to be
 *     exchanged by the caller, e.g. torch.distributed all_gather_object);
 *   nlinv_plan_connect: handles = world * 64 bytes in rank order (own entry ignored); opens them;
 *   nlinv_plan_connect_local: plans = the world plans of this job in rank order, all in this
 *     process (same or peer-accessible devices; tests and single-process drivers).
 * Requires the rank's coils to fit one fused K5 wave and one K4 chunk (ERR_SIZE at plan creation)
 * and world <= 8. All ranks must run the same sequence of calls (the exchanges are matched by
 * per-kind epoch counters). ERR_STATE if the plan is not a peer-memory plan or already connected. */
nlinv_status nlinv_plan_exchange_handle(nlinv_plan plan, unsigned char handle[64]);
nlinv_status nlinv_plan_connect(nlinv_plan plan, const unsigned char* handles);
nlinv_status nlinv_plan_connect_local(nlinv_plan plan, const nlinv_plan* plans);

/* Debug: how many thread-block clusters of the cluster-fused K2 -> K3 -> K4 pass (one cluster per
 * coil, DSMEM transposes) can be co-resident on the current device at grid size ng
 * (cudaOccupancyMaxActiveClusters); < 0 if that pass is not built for ng. Needs a device. */
int nlinv_debug_k234_clusters(int ng);

/* Micro-benchmark entry (the paper's axpy of Fig. 4): y = a x + y over n
 * floats (device pointers, n a multiple of 4, 16-byte aligned), enqueued on `stream`. ERR_ARG on NULL
 * pointers or a bad n. No plan needed. */
nlinv_status nlinv_debug_axpy(float a, const float* x, float* y, long long n, void* stream);

/* Number of kernels this library enqueued since plan creation (launch-count evidence). */
long long nlinv_plan_launch_count(nlinv_plan plan);

/* ---------------------------------------------------------------------------------------------
 * GPU gridding of radial spokes ("initial interpolation of the data
 * to the grid ... pre-processing step on the CPU", P:346 radial; reading R20). Frame f's spoke s
 * (theta = pi (s turns + f mod turns) / (spokes turns)) carries ng readout samples at r = i - ng/2;
 * sample (s, i) goes to the R12 cell of (r cos theta, r sin theta); a sampled cell gets the mean of
 * its samples in ascending (s, i) order. Raw samples: c32 [count][spokes][ng] (local coils).
 * ------------------------------------------------------------------------------------------- */

/* Build the per-phase cell lists (host, integer-exact, same rule as nlinv_radial_mask) and upload
 * them. Synchronises the device. ERR_STATE if a sample is within 1e-6 of a snap midpoint. */
nlinv_status nlinv_plan_set_trajectory(nlinv_plan plan, int spokes, int turns);

/* Convolution gridding instead (reading R22): separable Kaiser-Bessel window of `width` grid cells
 * (0 < width <= 8; beta <= 0 selects Beatty's value for oversampling 2). A sampled cell gets the
 * window-weighted mean of the samples within width/2 and the frame's P_k becomes real-valued,
 * P_k = sqrt(PSF), PSF = sum of the window weights (the operators then use P_k on the data and
 * P_k^2 in the normal operator). Host tables in fp64, weights stored in fp32. Synchronises. */
nlinv_status nlinv_plan_set_trajectory_kb(nlinv_plan plan, int spokes, int turns, double width, double beta);

/* Grid frame `frame` (phase frame mod turns): writes y[j][cell] for every sampled cell of P_k
 * (other cells untouched: only P_k y enters the method, R16) and sets the plan's P_k to that
 * frame's mask. raw: device [count][spokes][ng]; y: device [count][ng][ng]. Stream-ordered.
 * ERR_STATE before nlinv_plan_set_trajectory. */
nlinv_status nlinv_grid_radial(nlinv_plan plan, int frame, const nlinv_c32* raw, nlinv_c32* y, void* stream);

/* Real-time entry with raw radial samples (pinned host [count][spokes][ng]): H2D, GPU gridding,
 * reconstruction with the previous frame as prior (as nlinv_stream_frame), image to image_host
 * (host [n][n], may be NULL). Synchronises the stream before returning. */
nlinv_status nlinv_stream_frame_radial(nlinv_plan plan, const nlinv_c32* raw_host, int frame, int newton_steps,
                                       int cg_iters, nlinv_c32* image_host, void* stream);

/* ---------------------------------------------------------------------------------------------
 * PCA channel compression. PAPER P:241 (§3.2): "A principal component
 * analysis preprocessing step is applied before reconstruction to compress the 32 channels to
 * 8-12"; covariance C = sum_n y[n] y[n]^H (J x J), eigendecomposition, projection
 * y'_k = v_k^H y onto the top-J' eigenvectors (descending eigenvalues), each v_k scaled by a unit
 * phase so that its largest-magnitude component (first index on ties) is real-positive.
 * Channel data Y: device c32 [J][nsamp] (channel rows, any sample set: a full gridded frame or
 * its compact samples). A handle owns its workspace; not thread-safe; plan-independent.
 * ------------------------------------------------------------------------------------------- */
typedef struct nlinv_pca_s* nlinv_pca;

/* 1 <= J <= 32 channels (ERR_SIZE otherwise), 1 <= Jc <= J kept components (ERR_ARG). Allocates
 * on the current CUDA device (ERR_NOMEM). */
nlinv_status nlinv_pca_create(int J, int Jc, nlinv_pca* out);
nlinv_status nlinv_pca_destroy(nlinv_pca pca);

/* Fit: C (fp64, deterministic CTA-order reduction), Jacobi eigendecomposition (fp64), V. Enqueued
 * on `stream`, no host sync. Y: device [J][nsamp], nsamp >= 1. */
nlinv_status nlinv_pca_fit(nlinv_pca pca, const nlinv_c32* Y, long long nsamp, void* stream);

/* Host readback of the last fit (synchronises the device). Any output may be NULL.
 * V_host: c32 [J][Jc] row-major (V[j*Jc + k] = component j of v_k); eig_host: fp64 [J] descending;
 * energy: captured fraction sum_{k<Jc} lambda_k / sum_k lambda_k (negative rounding clipped to 0);
 * cov_host: fp64 [J][J][2] (re, im) covariance. ERR_STATE before any fit / set_matrix. */
nlinv_status nlinv_pca_result(nlinv_pca pca, nlinv_c32* V_host, double* eig_host, double* energy,
                              double* cov_host);

/* Use a given compression matrix (host c32 [J][Jc]) instead of a fit, e.g. one fitted on the
 * first frame of a stream. */
nlinv_status nlinv_pca_set_matrix(nlinv_pca pca, const nlinv_c32* V_host);

/* Apply: out[k][n] = sum_j conj(V[j][k]) Y[j][n] (channels summed in ascending order, fp32).
 * Y: device [J][nsamp]; out: device [Jc][nsamp], must not overlap Y (ERR_ARG). ERR_STATE before
 * any fit / set_matrix. Enqueued on `stream`. */
nlinv_status nlinv_pca_apply(nlinv_pca pca, const nlinv_c32* Y, long long nsamp, nlinv_c32* out, void* stream);

/* Last error message of this handle (never NULL) and its number of enqueued kernels. */
const char* nlinv_pca_last_error(nlinv_pca pca);
long long nlinv_pca_launch_count(nlinv_pca pca);

#ifdef __cplusplus
}
#endif
#endif /* NLINV_H_ */
