// Host side of libnlinv.so: the C ABI declared in include/nlinv.h.
//
// Owns the plan (workspace, tables, NCCL communicator, CUDA-graph cache) and drives the
// IRGNM / CG iteration of PAPER.md Eq. 3 by enqueuing the kernels of
// nlinv_kernels.cu. No arithmetic of the method runs here except the one-time tables
// (twiddles, w^{-1}) and the integer radial rasteriser, which are host setup.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nlinv.h"
#include "nlinv_kernels.cuh"

#ifdef NLINV_WITH_NCCL
#include <nccl.h>
#endif

using namespace nlv;

namespace {

thread_local std::string g_lib_error = "";

struct GraphKey {
  const void* frame = nullptr;
  const void* prior = nullptr;
  const void* xout = nullptr;
  const void* img = nullptr;
  const void* pw = nullptr;   // real-valued P_k buffer in use (KB gridding) or nullptr
  int K = -1, L = -1;
  cudaStream_t stream = nullptr;
  bool operator==(const GraphKey& o) const {
    return frame == o.frame && prior == o.prior && xout == o.xout && img == o.img && pw == o.pw && K == o.K &&
           L == o.L && stream == o.stream;
  }
};

}  // namespace

struct nlinv_plan_s {
  int ng = 0, n = 0, J = 0, rank = 0, world = 1, first = 0, count = 0;
  size_t N = 0, H = 0, Q = 0;
  nlinv_params prm{};
  int device = 0;
  std::string err;
  bool point_set = false;
  long long launches = 0;
  // tables
  float2* tw = nullptr;
  float* winv = nullptr;
  uint8_t* mask = nullptr;
  // workspace
  float2 *xref = nullptr, *dx = nullptr, *r = nullptr, *p = nullptr, *Ap = nullptr;
  float2 *tA = nullptr, *tB = nullptr, *c_omega = nullptr, *rho_omega = nullptr;
  float2 *S_all = nullptr, *S = nullptr, *S_sum = nullptr;   // per-coil terms; local sum; rank sum
  float *rss_all = nullptr, *rss = nullptr, *rss_sum = nullptr;
  int trace_mode = -1;                    // debug: column mode whose CTA timelines are recorded
  bool multi = false;                     // NCCL collective code path (world > 1 with an NCCL id, or NLINV_FORCE_NCCL=1)
  bool p2p = false;                       // peer-memory exchange (world > 1 without an NCCL id)
  XPeers xp{};                            // connected peers (xp.G == 0 until nlinv_plan_connect*)
  XPeers* xp_dev = nullptr;               // device copy of xp passed to the kernels (nullptr until connected)
  char* xwin = nullptr;                   // this rank's exchange window (IPC-exportable)
  std::vector<void*> ipc_open;            // peer windows opened through CUDA IPC
  bool fused = false;                     // fused K5 + CG + K1 pass, one grid barrier (k5cg_kernel, R19)
  int k5_rows = 0;                        // its CTA rows (>= J; the extra rows carry rho stripes only)
  bool k234 = false;                      // cluster-fused K2 -> K3 -> K4 in the fused CG loop (k234_kernel)
  bool cg1 = false;                       // unfused CG: one (grouped) scalar all-reduce per iteration (R19)
  unsigned* kbar = nullptr;               // its grid barrier
  CUtensorMap* tmaps = nullptr;           // device copies of the TMA tensor maps of r and dx (k5cg prefetch)
  double* kpart = nullptr;                // its dot partials
  unsigned long long* trace = nullptr;
  double *scal = nullptr, *partials = nullptr;
  unsigned* counter = nullptr;
  // host e2e staging (device side)
  float2 *h_frame = nullptr, *h_x = nullptr, *h_img = nullptr;
  // sampled-cell index list of P_k (nlinv_mask_indices, compact ingest)
  int *midx = nullptr, *mcount = nullptr, *mnnz = nullptr;
  float2* h_samples = nullptr;
  // radial trajectory (nlinv_plan_set_trajectory): per frame phase f mod turns, the sampled cells
  // (ascending), CSR starts, sample ids and P_k on the device
  int traj_spokes = 0, traj_turns = 0;
  std::vector<int*> tr_cells, tr_start, tr_sid;
  std::vector<uint8_t*> tr_mask;
  std::vector<int> tr_nnz;
  std::vector<float*> tr_wgt, tr_pw;   // KB gridding (R22): per-entry weights, sqrt(PSF) per cell
  const float* pw_active = nullptr;    // real-valued P_k of the current frame (nullptr = binary P_k)
  float* pw_buf = nullptr;             // fixed device copy of the frame's sqrt(PSF) (graph-stable pointer)
  float2* h_raw = nullptr;   // staging of host raw samples (nlinv_stream_frame_radial)
  void* slab = nullptr;      // one allocation for the per-iteration working set
  long long mnnz_host = -1;  // count of midx; -1 = index list stale (P_k changed)
  // graph cache
  GraphKey gkey;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;          // graph stream for callers on the legacy default stream
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  long long gkernels = 0;
  cudaStream_t last_stream = nullptr;
  int last_K = 0, last_L = 0;
  // streaming state (nlinv_stream_frame)
  bool stream_started = false;
  // per-kernel event profiling (nlinv_plan_set_profiling)
  struct ProfRec {
    const char* name;
    cudaEvent_t e0, e1;
  };
  bool prof = false;
  std::vector<ProfRec> prof_rec;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
#ifdef NLINV_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
};

namespace nlv {
void set_lib_error(const std::string& msg) { g_lib_error = msg; }   // pca.cu
}  // namespace nlv

static nlinv_status fail(nlinv_plan pl, nlinv_status s, const std::string& msg) {
  if (pl) pl->err = msg;
  g_lib_error = msg;
  return s;
}

#define CU(call)                                                                                \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return fail(pl, NLINV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

#ifdef NLINV_WITH_NCCL
#define NC(call)                                                                                \
  do {                                                                                          \
    ncclResult_t e_ = (call);                                                                   \
    if (e_ != ncclSuccess)                                                                      \
      return fail(pl, NLINV_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(e_));      \
  } while (0)
#endif

// ------------------------------------------------------------------ small public helpers
extern "C" void nlinv_params_default(nlinv_params* p) {
  if (!p) return;
  p->sob_a = 220.0f;
  p->sob_b = 32.0f;
  p->alpha0 = 1.0f;
  p->q = 1.0f / 3.0f;
  p->fov_full = 0;
  p->rank = 0;
  p->world = 1;
  p->nccl_id = nullptr;
}

extern "C" const char* nlinv_status_string(nlinv_status s) {
  switch (s) {
    case NLINV_OK: return "NLINV_OK";
    case NLINV_ERR_ARG: return "NLINV_ERR_ARG";
    case NLINV_ERR_SIZE: return "NLINV_ERR_SIZE";
    case NLINV_ERR_STATE: return "NLINV_ERR_STATE";
    case NLINV_ERR_CUDA: return "NLINV_ERR_CUDA";
    case NLINV_ERR_NCCL: return "NLINV_ERR_NCCL";
    case NLINV_ERR_NOMEM: return "NLINV_ERR_NOMEM";
    case NLINV_ERR_DIVERGED: return "NLINV_ERR_DIVERGED";
    case NLINV_ERR_NOT_BUILT: return "NLINV_ERR_NOT_BUILT";
  }
  return "NLINV_ERR_UNKNOWN";
}

extern "C" const char* nlinv_last_error(nlinv_plan plan) { return plan ? plan->err.c_str() : g_lib_error.c_str(); }

extern "C" const char* nlinv_build_info(void) {
#ifdef NLINV_WITH_NCCL
  return "libnlinv sm_100a nccl=1";
#else
  return "libnlinv sm_100a nccl=0";
#endif
}

extern "C" nlinv_status nlinv_get_unique_id(unsigned char id[128]) {
  nlinv_plan pl = nullptr;
  if (!id) return fail(pl, NLINV_ERR_ARG, "id is NULL");
#ifdef NLINV_WITH_NCCL
  ncclUniqueId uid;
  NC(ncclGetUniqueId(&uid));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &uid, 128);
  return NLINV_OK;
#else
  return fail(pl, NLINV_ERR_NOT_BUILT, "built without NCCL");
#endif
}

// ------------------------------------------------------------------ radial rasteriser (R12)
// Integer-exact: v is snapped to the 2^-20 grid, then rounded half away from zero.
static bool round_snapped(double v, long long* out) {
  const double f = v * 1048576.0;
  const double fr = f - std::floor(f);
  if (std::fabs(fr - 0.5) <= 1e-6) return false;  // too close to a snap midpoint
  const long long s = (long long)std::llround(f);
  const long long a = s < 0 ? -s : s;
  const long long qv = (a + (1LL << 19)) >> 20;
  *out = s < 0 ? -qv : qv;
  return true;
}

extern "C" nlinv_status nlinv_radial_mask(int nx, int ny, int spokes, int turns, int frame, uint8_t* out) {
  nlinv_plan pl = nullptr;
  if (!out) return fail(pl, NLINV_ERR_ARG, "out is NULL");
  if (nx != ny || nx < 2 || nx % 2) return fail(pl, NLINV_ERR_SIZE, "radial mask needs an even square grid");
  if (spokes < 1 || turns < 1 || frame < 0) return fail(pl, NLINV_ERR_ARG, "bad spokes/turns/frame");
  const int ng = nx;
  std::memset(out, 0, (size_t)ng * ng);
  const double denom = (double)spokes * (double)turns;
  for (int s = 0; s < spokes; ++s) {
    const double theta = M_PI * (double)(s * turns + (frame % turns)) / denom;
    const double ct = std::cos(theta), st = std::sin(theta);
    for (int i = 0; i < ng; ++i) {
      const double rr = (double)(i - ng / 2);
      long long kx, ky;
      if (!round_snapped(rr * ct, &kx) || !round_snapped(rr * st, &ky))
        return fail(pl, NLINV_ERR_STATE, "radial sample within 1e-6 of a snap midpoint");
      kx += ng / 2;
      ky += ng / 2;
      if (kx >= 0 && kx < ng && ky >= 0 && ky < ng) out[ky * ng + kx] = 1;
    }
  }
  return NLINV_OK;
}

// ------------------------------------------------------------------ radial trajectory + GPU gridding (f2, R20)
static nlinv_status traj_clear(nlinv_plan pl) {
  for (int* p : pl->tr_cells) cudaFree(p);
  for (int* p : pl->tr_start) cudaFree(p);
  for (int* p : pl->tr_sid) cudaFree(p);
  for (uint8_t* p : pl->tr_mask) cudaFree(p);
  for (float* p : pl->tr_wgt) cudaFree(p);
  for (float* p : pl->tr_pw) cudaFree(p);
  pl->tr_wgt.clear();
  pl->tr_pw.clear();
  pl->pw_active = nullptr;
  pl->tr_cells.clear();
  pl->tr_start.clear();
  pl->tr_sid.clear();
  pl->tr_mask.clear();
  pl->tr_nnz.clear();
  pl->traj_spokes = pl->traj_turns = 0;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_set_trajectory(nlinv_plan pl, int spokes, int turns) {
  if (!pl) return fail(pl, NLINV_ERR_ARG, "NULL plan");
  if (spokes < 1 || turns < 1 || turns > 64) return fail(pl, NLINV_ERR_ARG, "bad spokes/turns");
  CU(cudaDeviceSynchronize());
  traj_clear(pl);
  const int ng = pl->ng;
  const size_t N = pl->N;
  const double denom = (double)spokes * (double)turns;
  for (int f = 0; f < turns; ++f) {
    // cell of every sample by the R12 rule (same integer arithmetic as nlinv_radial_mask)
    std::vector<std::pair<int, int>> cs;   // (cell, sample id), sample ids ascending
    cs.reserve((size_t)spokes * ng);
    for (int sp = 0; sp < spokes; ++sp) {
      const double theta = M_PI * (double)(sp * turns + f) / denom;
      const double ct = std::cos(theta), st = std::sin(theta);
      for (int i = 0; i < ng; ++i) {
        const double rr = (double)(i - ng / 2);
        long long kx, ky;
        if (!round_snapped(rr * ct, &kx) || !round_snapped(rr * st, &ky)) {
          traj_clear(pl);
          return fail(pl, NLINV_ERR_STATE, "radial sample within 1e-6 of a snap midpoint");
        }
        kx += ng / 2;
        ky += ng / 2;
        if (kx >= 0 && kx < ng && ky >= 0 && ky < ng) cs.push_back({(int)(ky * ng + kx), sp * ng + i});
      }
    }
    std::stable_sort(cs.begin(), cs.end(), [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
      return a.first < b.first;
    });
    std::vector<int> cells, start, sid;
    std::vector<uint8_t> m(N, 0);
    for (size_t u = 0; u < cs.size(); ++u) {
      if (u == 0 || cs[u].first != cs[u - 1].first) {
        cells.push_back(cs[u].first);
        start.push_back((int)u);
        m[cs[u].first] = 1;
      }
      sid.push_back(cs[u].second);
    }
    start.push_back((int)cs.size());
    int *dc = nullptr, *ds = nullptr, *di = nullptr;
    uint8_t* dm = nullptr;
    CU(cudaMalloc((void**)&dc, sizeof(int) * (cells.size() + 1)));
    CU(cudaMalloc((void**)&ds, sizeof(int) * start.size()));
    CU(cudaMalloc((void**)&di, sizeof(int) * (sid.size() + 1)));
    CU(cudaMalloc((void**)&dm, N));
    pl->tr_cells.push_back(dc);
    pl->tr_start.push_back(ds);
    pl->tr_sid.push_back(di);
    pl->tr_mask.push_back(dm);
    pl->tr_nnz.push_back((int)cells.size());
    if (!cells.empty()) CU(cudaMemcpy(dc, cells.data(), sizeof(int) * cells.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ds, start.data(), sizeof(int) * start.size(), cudaMemcpyHostToDevice));
    if (!sid.empty()) CU(cudaMemcpy(di, sid.data(), sizeof(int) * sid.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dm, m.data(), N, cudaMemcpyHostToDevice));
  }
  pl->traj_spokes = spokes;
  pl->traj_turns = turns;
  return NLINV_OK;
}

// Kaiser-Bessel window (R22): I0 by its power series, Beatty's beta for oversampling 2 when beta <= 0
static double kb_i0(double z) {
  double term = 1.0, s = 1.0;
  const double q = 0.25 * z * z;
  for (int k = 1; term > 1e-17 * s; ++k) {
    term *= q / ((double)k * (double)k);
    s += term;
  }
  return s;
}
static double kb_h(double d, double width, double beta, double i0b) {
  const double u = 2.0 * d / width;
  if (std::fabs(u) > 1.0) return 0.0;
  return kb_i0(beta * std::sqrt(1.0 - u * u)) / i0b;
}

extern "C" nlinv_status nlinv_plan_set_trajectory_kb(nlinv_plan pl, int spokes, int turns, double width, double beta) {
  if (!pl) return fail(pl, NLINV_ERR_ARG, "NULL plan");
  if (spokes < 1 || turns < 1 || turns > 64) return fail(pl, NLINV_ERR_ARG, "bad spokes/turns");
  if (!(width > 0.0 && width <= 8.0)) return fail(pl, NLINV_ERR_ARG, "KB width must be in (0, 8] cells");
  if (beta <= 0.0) beta = M_PI * std::sqrt((width / 2.0) * (width / 2.0) * 2.25 - 0.8);
  CU(cudaDeviceSynchronize());
  traj_clear(pl);
  const int ng = pl->ng;
  const size_t N = pl->N;
  const double denom = (double)spokes * (double)turns, half = width / 2.0, c = (double)(ng / 2);
  const double i0b = kb_i0(beta);
  for (int f = 0; f < turns; ++f) {
    struct Ent { int cell, sid; double h; };
    std::vector<Ent> es;
    for (int sp = 0; sp < spokes; ++sp) {
      const double theta = M_PI * (double)(sp * turns + f) / denom;
      const double ct = std::cos(theta), st = std::sin(theta);
      for (int i = 0; i < ng; ++i) {
        const double rr = (double)(i - ng / 2);
        const double kx = c + rr * ct, ky = c + rr * st;
        for (long long gy = (long long)std::ceil(ky - half); gy <= (long long)std::floor(ky + half); ++gy) {
          const double hy = kb_h((double)gy - ky, width, beta, i0b);
          if (hy == 0.0 || gy < 0 || gy >= ng) continue;
          for (long long gx = (long long)std::ceil(kx - half); gx <= (long long)std::floor(kx + half); ++gx) {
            const double hx = kb_h((double)gx - kx, width, beta, i0b);
            if (hx == 0.0 || gx < 0 || gx >= ng) continue;
            es.push_back({(int)(gy * ng + gx), sp * ng + i, hx * hy});
          }
        }
      }
    }
    std::stable_sort(es.begin(), es.end(), [](const Ent& a, const Ent& b) { return a.cell < b.cell; });
    std::vector<int> cells, start, sid;
    std::vector<float> wgt, pw(N, 0.0f);
    std::vector<uint8_t> m(N, 0);
    double psf = 0.0;
    for (size_t u = 0; u < es.size(); ++u) {
      if (u == 0 || es[u].cell != es[u - 1].cell) {
        if (u > 0) pw[es[u - 1].cell] = (float)std::sqrt(psf);
        cells.push_back(es[u].cell);
        start.push_back((int)u);
        m[es[u].cell] = 1;
        psf = 0.0;
      }
      psf += es[u].h;
      sid.push_back(es[u].sid);
      wgt.push_back((float)es[u].h);
    }
    if (!es.empty()) pw[es.back().cell] = (float)std::sqrt(psf);
    start.push_back((int)es.size());
    int *dc = nullptr, *ds = nullptr, *di = nullptr;
    uint8_t* dm = nullptr;
    float *dw = nullptr, *dp = nullptr;
    CU(cudaMalloc((void**)&dc, sizeof(int) * (cells.size() + 1)));
    CU(cudaMalloc((void**)&ds, sizeof(int) * start.size()));
    CU(cudaMalloc((void**)&di, sizeof(int) * (sid.size() + 1)));
    CU(cudaMalloc((void**)&dw, sizeof(float) * (wgt.size() + 1)));
    CU(cudaMalloc((void**)&dp, sizeof(float) * N));
    CU(cudaMalloc((void**)&dm, N));
    pl->tr_cells.push_back(dc);
    pl->tr_start.push_back(ds);
    pl->tr_sid.push_back(di);
    pl->tr_wgt.push_back(dw);
    pl->tr_pw.push_back(dp);
    pl->tr_mask.push_back(dm);
    pl->tr_nnz.push_back((int)cells.size());
    if (!cells.empty()) CU(cudaMemcpy(dc, cells.data(), sizeof(int) * cells.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ds, start.data(), sizeof(int) * start.size(), cudaMemcpyHostToDevice));
    if (!sid.empty()) CU(cudaMemcpy(di, sid.data(), sizeof(int) * sid.size(), cudaMemcpyHostToDevice));
    if (!wgt.empty()) CU(cudaMemcpy(dw, wgt.data(), sizeof(float) * wgt.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dp, pw.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dm, m.data(), N, cudaMemcpyHostToDevice));
  }
  pl->traj_spokes = spokes;
  pl->traj_turns = turns;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_grid_radial(nlinv_plan pl, int frame, const nlinv_c32* raw, nlinv_c32* y, void* stream) {
  if (!pl || !raw || !y || frame < 0) return fail(pl, NLINV_ERR_ARG, "bad argument to nlinv_grid_radial");
  if (pl->traj_turns == 0) return fail(pl, NLINV_ERR_STATE, "nlinv_grid_radial before nlinv_plan_set_trajectory");
  cudaStream_t s = (cudaStream_t)stream;
  const int f = frame % pl->traj_turns;
  const int nraw = pl->traj_spokes * pl->ng;
  CU(cudaMemcpyAsync(pl->mask, pl->tr_mask[f], pl->N, cudaMemcpyDeviceToDevice, s));
  pl->mnnz_host = -1;
  const bool kb = !pl->tr_wgt.empty();
  if (kb) {   // KB gridding: the frame's real-valued P_k (R22), copied to a graph-stable buffer
    if (!pl->pw_buf) CU(cudaMalloc((void**)&pl->pw_buf, sizeof(float) * pl->N));
    CU(cudaMemcpyAsync(pl->pw_buf, pl->tr_pw[f], sizeof(float) * pl->N, cudaMemcpyDeviceToDevice, s));
    pl->pw_active = pl->pw_buf;
  } else {
    pl->pw_active = nullptr;
  }
  CU(launch_grid_radial(reinterpret_cast<const float2*>(raw), pl->J, nraw, pl->tr_cells[f], pl->tr_start[f],
                        pl->tr_sid[f], kb ? pl->tr_wgt[f] : nullptr, pl->tr_nnz[f], pl->N,
                        reinterpret_cast<float2*>(y), s));
  pl->launches += 1;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_coil_partition(int ncoils, int world, int rank, int* first, int* count) {
  nlinv_plan pl = nullptr;
  if (!first || !count) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (ncoils < 1 || world < 1 || world > ncoils || rank < 0 || rank >= world)
    return fail(pl, NLINV_ERR_ARG, "bad ncoils/world/rank");
  const int base = ncoils / world, rem = ncoils % world;
  *count = base + (rank < rem ? 1 : 0);
  *first = rank * base + (rank < rem ? rank : rem);
  return NLINV_OK;
}

// ------------------------------------------------------------------ plan
static void plan_free(nlinv_plan pl) {
  if (!pl) return;
  for (int* p : pl->tr_cells) cudaFree(p);
  for (int* p : pl->tr_start) cudaFree(p);
  for (int* p : pl->tr_sid) cudaFree(p);
  for (uint8_t* p : pl->tr_mask) cudaFree(p);
  for (float* p : pl->tr_wgt) cudaFree(p);
  for (float* p : pl->tr_pw) cudaFree(p);
  cudaFree(pl->h_raw);
  cudaFree(pl->pw_buf);
  for (void* w : pl->ipc_open) cudaIpcCloseMemHandle(w);
  cudaFree(pl->xwin);
  if (pl->slab) {   // tA, tB, dx, r, p, c_omega live in one slab
    cudaFree(pl->slab);
    pl->tA = pl->tB = pl->dx = pl->r = pl->p = pl->c_omega = nullptr;
  }
  void* ptrs[] = {pl->tw, pl->winv, pl->mask, pl->xref, pl->dx, pl->r, pl->p, pl->Ap, pl->tA, pl->tB,
                  pl->c_omega, pl->rho_omega, pl->S_all, pl->S, pl->S_sum, pl->rss_all, pl->rss, pl->rss_sum,
                  pl->kbar, pl->kpart, pl->tmaps, pl->xp_dev, pl->scal, pl->partials,
                  pl->counter, pl->h_frame, pl->h_x, pl->h_img, pl->midx, pl->mcount, pl->mnnz, pl->h_samples};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
  if (pl->gev_in) cudaEventDestroy(pl->gev_in);
  if (pl->gev_out) cudaEventDestroy(pl->gev_out);
  if (pl->gstream) cudaStreamDestroy(pl->gstream);
  for (cudaEvent_t e : pl->ev_pool) cudaEventDestroy(e);
#ifdef NLINV_WITH_NCCL
  if (pl->comm) ncclCommDestroy(pl->comm);
#endif
  delete pl;
}

// TMA descriptors of the chat blocks [J][ng][ng] (8-byte elements) of r and dx: box = one fused-pass
// column tile (CW columns) x up to 256 rows x one coil. false if the driver entry point is missing.
static bool make_tile_maps(int ng, int J, float2* r_chat, float2* dx_chat, float2* p_chat, CUtensorMap out[3]) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int cw = ng / col_tiles(ng);
  const cuuint64_t dims[3] = {(cuuint64_t)ng, (cuuint64_t)ng, (cuuint64_t)J};
  const cuuint64_t strides[2] = {(cuuint64_t)ng * 8, (cuuint64_t)ng * ng * 8};
  const cuuint32_t box[3] = {(cuuint32_t)cw, (cuuint32_t)(ng <= 256 ? ng : (ng % 256 == 0 ? 256 : 192)), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  float2* bases[3] = {r_chat, dx_chat, p_chat};
  for (int k = 0; k < 3; ++k) {
    if (enc(&out[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bases[k], dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

extern "C" nlinv_status nlinv_plan_create(int nx, int ny, int ncoils, const uint8_t* mask, const nlinv_params* p,
                                          nlinv_plan* out) {
  nlinv_plan pl = nullptr;
  if (!out || !mask) return fail(pl, NLINV_ERR_ARG, "NULL argument to nlinv_plan_create");
  *out = nullptr;
  if (nx != ny) return fail(pl, NLINV_ERR_SIZE, "nx != ny (square grids only)");
  if (!supported_ng(nx)) return fail(pl, NLINV_ERR_SIZE, "unsupported grid size " + std::to_string(nx));
  if (ncoils < 1 || ncoils > 256) return fail(pl, NLINV_ERR_SIZE, "ncoils must be in [1, 256]");
  nlinv_params prm;
  nlinv_params_default(&prm);
  if (p) prm = *p;
  if (prm.world < 1 || prm.rank < 0 || prm.rank >= prm.world) return fail(pl, NLINV_ERR_ARG, "bad rank/world");
  if (prm.world > ncoils) return fail(pl, NLINV_ERR_SIZE, "more ranks than coils");
  if (!(prm.q > 0.0f) || !(prm.alpha0 > 0.0f)) return fail(pl, NLINV_ERR_ARG, "alpha0 and q must be > 0");
#ifndef NLINV_WITH_NCCL
  if (prm.world > 1 && prm.nccl_id) return fail(pl, NLINV_ERR_NOT_BUILT, "built without NCCL");
#endif
  if (prm.world > kMaxRanks && !prm.nccl_id)
    return fail(pl, NLINV_ERR_SIZE, "the peer-memory exchange supports at most 8 ranks (one node)");
  if (prm.fov_full) return fail(pl, NLINV_ERR_ARG, "fov_full is an oracle-only test mode (Omega pruning is structural)");
  {
    int dev = -1;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return fail(pl, NLINV_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(de));
  }

  pl = new nlinv_plan_s();
  pl->prm = prm;
  pl->prm.nccl_id = nullptr;
  pl->ng = nx;
  pl->n = nx / 2;
  pl->N = (size_t)nx * nx;
  pl->H = (size_t)pl->n * nx;
  pl->Q = (size_t)pl->n * pl->n;
  pl->rank = prm.rank;
  pl->world = prm.world;
  {
    // multi-GPU code path (coil-sum and scalar all-reduces through NCCL, unfused CG): world > 1,
    // or NLINV_FORCE_NCCL=1 on one GPU (a one-rank communicator: the collective plumbing is then
    // exercised and parity-tested on a single device)
    const char* fn = std::getenv("NLINV_FORCE_NCCL");
#ifdef NLINV_WITH_NCCL
    pl->multi = (prm.world > 1 && prm.nccl_id != nullptr) || (prm.world == 1 && fn && fn[0] == '1');
#else
    pl->multi = false;
    (void)fn;
#endif
    pl->p2p = prm.world > 1 && !pl->multi;
  }
  nlinv_coil_partition(ncoils, prm.world, prm.rank, &pl->first, &pl->count);
  pl->J = pl->count;
  if ((long long)col_tiles(nx) * (pl->J + 1) > kMaxRedBlocks) {
    plan_free(pl);
    return fail(nullptr, NLINV_ERR_SIZE, "too many local coils for this grid");
  }
  cudaGetDevice(&pl->device);

  const size_t N = pl->N, nb = 1 + (size_t)pl->J;
  auto alloc = [&](void** ptr, size_t bytes) -> bool { return cudaMalloc(ptr, bytes) == cudaSuccess; };
  bool ok = true;
  ok &= alloc((void**)&pl->tw, sizeof(float2) * nx);
  ok &= alloc((void**)&pl->winv, sizeof(float) * N);
  ok &= alloc((void**)&pl->mask, N);
  ok &= alloc((void**)&pl->xref, sizeof(float2) * N * nb);
  // The per-CG-iteration working set (T intermediates, c|Omega, r, p, dx: ~65 MB at C2) is one
  // slab. (An L2-persisting access-policy window over it was measured within noise at C2, +0.6 %:
  // the passes are not DRAM bound; not kept.)
  {
    const size_t b_t = sizeof(float2) * pl->H * pl->J, b_v = sizeof(float2) * N * nb, b_c = sizeof(float2) * pl->Q * pl->J;
    const size_t tot_b = 2 * b_t + 3 * b_v + b_c;
    if (alloc(&pl->slab, tot_b)) {
      char* b = (char*)pl->slab;
      pl->tA = (float2*)b;
      pl->tB = (float2*)(b + b_t);
      pl->r = (float2*)(b + 2 * b_t);
      pl->p = (float2*)(b + 2 * b_t + b_v);
      pl->dx = (float2*)(b + 2 * b_t + 2 * b_v);
      pl->c_omega = (float2*)(b + 2 * b_t + 3 * b_v);
    } else {
      ok &= alloc((void**)&pl->dx, b_v);
      ok &= alloc((void**)&pl->r, b_v);
      ok &= alloc((void**)&pl->p, b_v);
      ok &= alloc((void**)&pl->tA, b_t);
      ok &= alloc((void**)&pl->tB, b_t);
      ok &= alloc((void**)&pl->c_omega, b_c);
    }
  }
  ok &= alloc((void**)&pl->Ap, sizeof(float2) * N * nb);
  ok &= alloc((void**)&pl->rho_omega, sizeof(float2) * pl->Q);
  ok &= alloc((void**)&pl->S, sizeof(float2) * pl->Q);
  ok &= alloc((void**)&pl->S_all, sizeof(float2) * pl->Q * pl->J);
  ok &= alloc((void**)&pl->rss_all, sizeof(float) * pl->Q * pl->J);
  if (pl->multi) {
    ok &= alloc((void**)&pl->rss, sizeof(float) * pl->Q);
    ok &= alloc((void**)&pl->S_sum, sizeof(float2) * pl->Q);
    ok &= alloc((void**)&pl->rss_sum, sizeof(float) * pl->Q);
  }
  {
    // single-reduction unfused CG: default where a reduction is a collective (multi-GPU path); on
    // one GPU the r update is cheaper as its own pass (measured), NLINV_CG1=1 forces it there
    const char* c1 = std::getenv("NLINV_CG1");
    pl->cg1 = c1 ? (c1[0] == '1') : pl->multi;
    // fused K5 + CG + K1 with one grid barrier (world == 1, the K5 grid fits one co-resident wave);
    // NLINV_FUSE_K5=0 forces the unfused passes
    const char* fk = std::getenv("NLINV_FUSE_K5");
    pl->fused = !pl->multi && !(fk && fk[0] == '0') && k5cg_fusable(nx, pl->J);
    // cluster-fused K2 -> K3 -> K4 (DSMEM transposes) inside the fused CG loop: opt-in (NLINV_K234=1).
    // Measured on B200 at C2 it is slower than the three PDL-chained passes (45.5 vs 40.4 us per
    // iteration, eager events): with 12 coils x 12-CTA clusters on 148 SMs some SMs host two CTAs
    // and every cluster barrier waits for them.
    const char* kc = std::getenv("NLINV_K234");
    pl->k234 = pl->fused && (kc && kc[0] == '1') && k234_supported(nx);
    if (pl->fused) {
      pl->k5_rows = k5cg_rows(nx, pl->J);
      ok &= alloc((void**)&pl->kbar, sizeof(unsigned) * 4);
      ok &= alloc((void**)&pl->kpart, sizeof(double) * 10 * kMaxRedBlocks);   // 8 dots + 2 <r_{i+1},r_{i+1}>
      // TMA tile prefetch of r / dx in the fused pass (NLINV_TMA=0: cp.async instead)
      const char* tm = std::getenv("NLINV_TMA");
      if (ok && !(tm && tm[0] == '0')) {
        CUtensorMap h[3];
        if (make_tile_maps(nx, pl->J, pl->r + N, pl->dx + N, pl->p + N, h)) {
          ok &= alloc((void**)&pl->tmaps, sizeof(h));
          ok &= ok && cudaMemcpy(pl->tmaps, h, sizeof(h), cudaMemcpyHostToDevice) == cudaSuccess;
        }
      }
    }
  }
  if (pl->p2p) {
    // the peer-memory path runs the fused CG pass on every rank with one coil-sum plane per rank
    if (!pl->fused || k4_planes(nx, pl->J) != 1) {
      plan_free(pl);
      return fail(nullptr, NLINV_ERR_SIZE, "peer-memory exchange: the rank's coils do not fit one fused wave / one K4 chunk");
    }
    ok &= alloc((void**)&pl->xwin, xwin_bytes(pl->Q));
    ok &= alloc((void**)&pl->rss_sum, sizeof(float) * pl->Q);
    ok &= preload_kernels(nx) == cudaSuccess;
  }
  ok &= alloc((void**)&pl->scal, sizeof(double) * SC_TOTAL);
  ok &= alloc((void**)&pl->partials, sizeof(double) * 8 * kMaxRedBlocks);
  ok &= alloc((void**)&pl->counter, sizeof(unsigned) * 4);
  if (!ok) {
    plan_free(pl);
    cudaGetLastError();
    return fail(nullptr, NLINV_ERR_NOMEM, "device allocation failed");
  }
  // one-time tables in fp64, rounded to fp32 (R2): the inter-pass twiddles e^{-2 pi i m / ng} of every
  // Stockham pass p >= 1 in the pass's [r - 1][k] block (m = k r ng / (NS R), fft.cuh tw_base), w^{-1}(k)
  std::vector<float2> tw(nx, make_float2(0.f, 0.f));
  {
    int R[4] = {1, 1, 1, 1};
    const int np = fft_radices(nx, R);
    size_t off = 0;
    int NS = R[0];
    for (int p = 1; p < np; ++p) {
      for (int r = 1; r < R[p]; ++r)
        for (int k = 0; k < NS; ++k) {
          const long long m = (long long)k * r * (nx / (NS * R[p]));
          const double ang = 2.0 * M_PI * (double)m / (double)nx;
          tw[off + (size_t)(r - 1) * NS + k] = make_float2((float)std::cos(ang), (float)(-std::sin(ang)));
        }
      off += (size_t)NS * (R[p] - 1);
      NS *= R[p];
    }
    if (off > (size_t)nx) {
      plan_free(pl);
      return fail(nullptr, NLINV_ERR_SIZE, "twiddle table exceeds ng entries");
    }
  }
  std::vector<float> wi(N);
  const double a = prm.sob_a, b = prm.sob_b;
  for (int y = 0; y < nx; ++y)
    for (int x = 0; x < nx; ++x) {
      const double ky = (double)(y - nx / 2) / nx, kx = (double)(x - nx / 2) / nx;
      wi[(size_t)y * nx + x] = (float)std::pow(1.0 + a * (kx * kx + ky * ky), -0.5 * b);
    }
  std::vector<uint8_t> m8(N);
  for (size_t i = 0; i < N; ++i) m8[i] = mask[i] ? 1 : 0;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaMemcpy(pl->tw, tw.data(), sizeof(float2) * nx, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(pl->winv, wi.data(), sizeof(float) * N, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(pl->mask, m8.data(), N, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(pl->scal, 0, sizeof(double) * SC_TOTAL);
  if (e == cudaSuccess) e = cudaMemset(pl->counter, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess && pl->kbar) e = cudaMemset(pl->kbar, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess && pl->xwin) e = cudaMemset(pl->xwin, 0, xwin_bytes(pl->Q));
  if (e == cudaSuccess && pl->xwin) e = cudaDeviceSynchronize();   // zeroed flags before any peer looks
  if (e != cudaSuccess) {
    std::string msg = std::string("plan upload: ") + cudaGetErrorString(e);
    plan_free(pl);
    return fail(nullptr, NLINV_ERR_CUDA, msg);
  }
#ifdef NLINV_WITH_NCCL
  if (pl->multi) {
    ncclUniqueId uid;
    ncclResult_t r = ncclSuccess;
    if (pl->world > 1) std::memcpy(&uid, p->nccl_id, 128);
    else r = ncclGetUniqueId(&uid);   // NLINV_FORCE_NCCL=1: one-rank communicator (test mode)
    if (r == ncclSuccess) r = ncclCommInitRank(&pl->comm, pl->world, uid, pl->rank);
    if (r != ncclSuccess) {
      std::string msg = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      pl->comm = nullptr;
      plan_free(pl);
      return fail(nullptr, NLINV_ERR_NCCL, msg);
    }
  }
#endif
  *out = pl;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_set_mask(nlinv_plan pl, const uint8_t* mask_host) {
  if (!pl || !mask_host) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  std::vector<uint8_t> m8(pl->N);
  for (size_t i = 0; i < pl->N; ++i) m8[i] = mask_host[i] ? 1 : 0;
  // the previous frame's work (possibly on a non-blocking stream) may still read P_k
  if (pl->last_stream) CU(cudaStreamSynchronize(pl->last_stream));
  if (pl->gstream) CU(cudaStreamSynchronize(pl->gstream));
  CU(cudaMemcpy(pl->mask, m8.data(), pl->N, cudaMemcpyHostToDevice));
  pl->mnnz_host = -1;
  pl->pw_active = nullptr;   // a binary P_k replaces any KB weights
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_set_mask_device(nlinv_plan pl, const uint8_t* mask_dev, void* stream) {
  if (!pl || !mask_dev) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  CU(cudaMemcpyAsync(pl->mask, mask_dev, pl->N, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  pl->mnnz_host = -1;
  pl->pw_active = nullptr;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_local_coils(nlinv_plan pl, int* first, int* count) {
  if (!pl || !first || !count) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  *first = pl->first;
  *count = pl->count;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_destroy(nlinv_plan pl) {
  if (!pl) return NLINV_OK;
  cudaDeviceSynchronize();
  plan_free(pl);
  return NLINV_OK;
}

extern "C" long long nlinv_plan_launch_count(nlinv_plan pl) { return pl ? pl->launches : -1; }

// ------------------------------------------------------------------ enqueue helpers
namespace {

const char* kColNames[] = {"col_ifft_w", "col_ifft_w_cg", "col_fwdp", "col_psf", "col_resadj", "col_adj1",
                           "col_fft_w_normal", "col_fft_w_rhs", "col_fft_w_adj", "col_k5cg"};
const char* kRowNames[] = {"row_setpoint", "row_setpoint_fwd", "row_rss", "row_k2", "row_k4"};

struct Enq {
  nlinv_plan pl;
  cudaStream_t s;
  long long kernels = 0;

  // launch one kernel; with profiling on, bracket it with events on its own stream
  template <class F>
  nlinv_status kern(const char* name, F&& launch) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (pl->prof) {
      e0 = pl->event();
      cudaEventRecord(e0, s);
    }
    cudaError_t e = launch();
    if (pl->prof) {
      e1 = pl->event();
      cudaEventRecord(e1, s);
      pl->prof_rec.push_back({name, e0, e1});
    }
    ++kernels;
    if (e != cudaSuccess) return fail(pl, NLINV_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
    return NLINV_OK;
  }
  nlinv_status col(int mode, ColArgs a) {
    // the fused K5 + CG pass is traced at CG iteration 1 only (a steady-state K5 -> CG -> K1 launch)
    const bool fused = mode == CK_K5CG;
    a.trace = (pl->trace_mode == mode && (!fused || (a.iter == 1 && a.fuse_k1))) ? pl->trace : nullptr;
    a.winv = pl->winv;
    a.mask = pl->mask;
    a.pw = pl->pw_active;
    a.scal = pl->scal;
    a.scal_w = pl->scal;
    a.counter = pl->counter;
    a.J = pl->J;
    a.xp = pl->xp_dev;
    const char* name = kColNames[mode];
    if (mode == CK_FFT_W_RHS && a.fuse_k1) name = "col_rhs_k1";
    if (mode == CK_K5CG) name = a.fuse_k1 ? "col_k5_cg_k1" : "col_k5_newton";
    return kern(name, [&] { return launch_col(pl->ng, mode, a, pl->tw, s); });
  }
  nlinv_status row(int mode, RowArgs a) {
    a.J = pl->J;
    if (mode == RK_K4) a.xp = pl->xp_dev;
    a.c_omega = pl->c_omega;
    a.rho_omega = pl->rho_omega;
    return kern(kRowNames[mode], [&] { return launch_row(pl->ng, mode, a, pl->tw, s); });
  }
  VecArgs vec() const {
    VecArgs v{};
    v.scal = pl->scal;
    v.scal_w = pl->scal;
    v.partials = pl->partials;
    v.counter = pl->counter;
    v.nrho = (long long)pl->N;
    v.ntot = (long long)pl->N * (1 + pl->J);
    return v;
  }
  // a stream operation that is not a kernel (memcpy)
  nlinv_status check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) return fail(pl, NLINV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return NLINV_OK;
  }
  // all-reduce (sum) over the coil shards; in place when src == dst. No-op for world == 1.
  nlinv_status allreduce_f(const float* src, float* dst, size_t count) {
    if (!pl->multi) return NLINV_OK;
#ifdef NLINV_WITH_NCCL
    NC(ncclAllReduce(src, dst, count, ncclFloat, ncclSum, pl->comm, s));
#endif
    return NLINV_OK;
  }
  nlinv_status allreduce_scalar(int slot) { return allreduce_scalars(slot, 1); }
  // several single-double all-reduces aggregated into one NCCL launch (ncclGroupStart/End)
  nlinv_status allreduce_group(const int* slots, int n) {
    if (!pl->multi) return NLINV_OK;
#ifdef NLINV_WITH_NCCL
    NC(ncclGroupStart());
    for (int k = 0; k < n; ++k)
      NC(ncclAllReduce(pl->scal + slots[k], pl->scal + slots[k], 1, ncclDouble, ncclSum, pl->comm, s));
    NC(ncclGroupEnd());
#endif
    return NLINV_OK;
  }
  nlinv_status allreduce_scalars(int slot, int count) {
    if (!pl->multi) return NLINV_OK;
#ifdef NLINV_WITH_NCCL
    NC(ncclAllReduce(pl->scal + slot, pl->scal + slot, count, ncclDouble, ncclSum, pl->comm, s));
#endif
    return NLINV_OK;
  }
};

#define TRY(x)                     \
  do {                             \
    nlinv_status st_ = (x);        \
    if (st_ != NLINV_OK) return st_; \
  } while (0)

// c_j on Omega and rho|Omega of the point x. fwd_out != NULL: also the first
// half of F(x) (row FFT of rho c_j) into fwd_out.
// t_ready: tA already holds the column pass of x (the previous fused Newton update folded it in).
nlinv_status enq_set_point(Enq& q, const float2* x, float2* fwd_out, bool t_ready = false) {
  nlinv_plan pl = q.pl;
  ColArgs ca{};
  ca.src = x + pl->N;
  ca.out = pl->tA;
  if (!t_ready) TRY(q.col(CK_IFFT_W, ca));
  RowArgs ra{};
  ra.in = pl->tA;
  ra.xrho = x;
  ra.out = fwd_out;
  TRY(q.row(fwd_out ? RK_SETPOINT_FWD : RK_SETPOINT, ra));
  return NLINV_OK;
}

// tB := row-FFT half of DF(dx) at the cached point (K1, K2)
nlinv_status enq_derivative_head(Enq& q, const float2* dx, bool cg_fused, int iter) {
  nlinv_plan pl = q.pl;
  ColArgs ca{};
  ca.out = pl->tA;
  if (cg_fused) {
    ca.r = pl->r + pl->N;
    ca.p = pl->p + pl->N;
    ca.dx = pl->dx + pl->N;
    ca.rho_r = pl->r;
    ca.rho_p = pl->p;
    ca.rho_dx = pl->dx;
    ca.iter = iter;
    if (pl->cg1) {   // r -= gamma A p of the previous iteration happens here (R19)
      ca.cg1 = 1;
      ca.src2 = pl->Ap + pl->N;
      ca.rho_a = pl->Ap;
    }
    TRY(q.col(CK_IFFT_W_CG, ca));
  } else {
    ca.src = dx + pl->N;
    TRY(q.col(CK_IFFT_W, ca));
  }
  RowArgs ra{};
  ra.in = pl->tA;
  ra.out = pl->tB;
  ra.prho = dx;
  TRY(q.row(RK_K2, ra));
  return NLINV_OK;
}

// K4 on tA -> tB and the per-coil terms conj(c_j) u_j; for world > 1 the local coil sum is
// all-reduced over ranks (the block-wise all-reduce of P:246 / P:289, out of place).
nlinv_status enq_k4_allreduce(Enq& q) {
  nlinv_plan pl = q.pl;
  RowArgs ra{};
  ra.in = pl->tA;
  ra.out = pl->tB;
  ra.S = pl->S_all;   // one plane per K4 coil chunk
  TRY(q.row(RK_K4, ra));   // peer exchange: K4 writes its plane into the window and publishes it
  if (pl->multi) {
    const int np = k4_planes(pl->ng, pl->J);
    TRY(q.kern("coil_sum", [&] { return launch_coil_sum(pl->ng, pl->S_all, np, pl->S, q.s); }));
    TRY(q.allreduce_f((const float*)pl->S, (float*)pl->S_sum, 2 * pl->Q));
  }
  return NLINV_OK;
}

// the coil-sum planes the rho slices add up (chunk planes in order, or the rank-summed plane)
void set_S(nlinv_plan pl, ColArgs& c) {
  if (pl->multi) {
    c.S = pl->S_sum;
    c.nS = 1;
  } else {
    c.S = pl->S_all;
    c.nS = k4_planes(pl->ng, pl->J);
  }
}

// out = (DF^H DF + alpha) dx; with_cg: the CG-fused variant on the plan's p (iteration iter)
nlinv_status enq_normal(Enq& q, float alpha, const float2* dx, float2* out, bool cg, int iter, int last_iter = -1) {
  nlinv_plan pl = q.pl;
  TRY(enq_derivative_head(q, dx, cg, iter));
  ColArgs ca{};
  ca.in = pl->tB;
  ca.out = pl->tA;
  TRY(q.col(CK_PSF, ca));
  TRY(enq_k4_allreduce(q));
  ColArgs cb{};
  cb.in = pl->tB;
  cb.src2 = dx + pl->N;
  cb.out = out + pl->N;
  set_S(pl, cb);
  cb.rho_a = dx;
  cb.rho_out = out;
  cb.alpha = alpha;
  cb.partials = cg ? pl->partials : nullptr;
  cb.out_slot = SC_PAP_CHAT + iter;
  cb.out_slot_rho = SC_PAP_RHO + iter;
  cb.iter = iter;
  const bool cg1 = cg && pl->cg1;
  if (cg1) {   // also <r,Ap>, <Ap,Ap>, <r,r> for the single reduction (R19)
    cb.cg1 = 1;
    cb.r = pl->r + pl->N;
    cb.rho_r = pl->r;
  }
  TRY(q.col(CK_FFT_W_NORMAL, cb));
  if (cg1) {   // ONE grouped all-reduce of the four chat parts (the rho parts are replicated)
    const int slots[4] = {SC_PAP_CHAT + iter, SC_RAP_CHAT + iter, SC_AA_CHAT + iter, SC_RR_CHAT + iter};
    TRY(q.allreduce_group(slots, 4));
  } else if (cg) {
    TRY(q.allreduce_scalar(SC_PAP_CHAT + iter));   // chat part; the rho part is replicated
  }
  return NLINV_OK;
}

// peer exchange at the end of a frame: ||P y - F(x_n)||^2 of every Newton step summed over the
// ranks (SC_RES slots, in place) and, with rss_out, the RSS plane summed over the ranks
nlinv_status enq_xchg_frame(Enq& q, int K, float* rss_out) {
  nlinv_plan pl = q.pl;
  XchgArgs xa{};
  xa.xp = pl->xp;
  xa.scal = pl->scal;
  xa.nsum = K < 64 ? K : 64;
  xa.nr0 = 0;
  for (int n = 0; n < xa.nsum; ++n) xa.src[n] = xa.dst[n] = SC_RES + n;
  xa.rss_out = rss_out;
  xa.Q = (int)pl->Q;
  return q.kern("xchg", [&] { return launch_xchg(xa, q.s); });
}

// the whole frame: K Newton steps of L CG iterations on x (in place)
nlinv_status enq_reconstruct(Enq& q, const float2* frame, const float2* prior, int K, int L, float2* x,
                             float2* img) {
  nlinv_plan pl = q.pl;
  const size_t N = pl->N, tot = N * (1 + pl->J);
  if (prior) {
    if (prior != pl->xref)
      TRY(q.check(cudaMemcpyAsync(pl->xref, prior, tot * sizeof(float2), cudaMemcpyDeviceToDevice, q.s), "copy prior"));
    if (prior != x)
      TRY(q.check(cudaMemcpyAsync(x, prior, tot * sizeof(float2), cudaMemcpyDeviceToDevice, q.s), "copy prior"));
  } else {
    TRY(q.kern("init_x", [&] { return launch_init_x(pl->xref, (long long)N, (long long)tot, q.s); }));
    TRY(q.kern("init_x", [&] { return launch_init_x(x, (long long)N, (long long)tot, q.s); }));
  }
  double alpha_d = pl->prm.alpha0;
  bool sp_ready = false;   // tA holds the set-point column pass of x (folded into the fused Newton update)
  for (int nstep = 0; nstep < K; ++nstep, alpha_d *= pl->prm.q) {
    const float alpha = (float)alpha_d;
    // set point + forward head
    TRY(enq_set_point(q, x, pl->tB, sp_ready));
    sp_ready = false;
    // residual r = P(y - F x) and the adjoint head on it (Table 1 rows F and DF^H)
    ColArgs ca{};
    ca.in = pl->tB;
    ca.out = pl->tA;
    ca.y = frame;
    ca.partials = pl->partials;
    ca.out_slot = SC_RES + nstep;
    TRY(q.col(CK_RESADJ, ca));
    TRY(q.allreduce_scalar(SC_RES + nstep));
    TRY(enq_k4_allreduce(q));
    // rhs b = DF^H r - alpha (x - x_ref); r = p = b (CG start, dx = 0)
    ColArgs cb{};
    cb.in = pl->tB;
    cb.src = x + N;
    cb.src2 = pl->xref + N;
    cb.r = pl->r + N;
    cb.p = pl->p + N;
    cb.alpha = alpha;
    cb.partials = pl->partials;
    cb.out_slot = SC_RR_CHAT + 0;
    cb.out_slot_rho = SC_RR_RHO + 0;
    set_S(pl, cb);
    cb.rho_a = x;
    cb.rho_b = pl->xref;
    cb.rho_r = pl->r;
    cb.rho_p = pl->p;
    if (pl->fused) {  // K1 of CG iteration 0 (p_0 = b) folded into the rhs pass
      cb.fuse_k1 = 1;
      cb.t1 = pl->tA;
    }
    TRY(q.col(CK_FFT_W_RHS, cb));
    TRY(q.allreduce_scalar(SC_RR_CHAT + 0));
    if (pl->fused) {
      // CG, fused form: per iteration K2, K3, K4 and one cooperative pass that does K5,
      // gamma, r -= gamma Ap, <r,r>, beta and K1 of the next iteration (or the Newton update)
      float2* pc = pl->p;
      for (int it = 0; it < L; ++it) {
        ColArgs c5{};
        if (pl->k234) {   // K2 -> K3 -> K4, one cluster per coil: T1 (tA) -> T4 (tB) + per-coil S planes
          RowArgs ra{};
          ra.in = pl->tA;
          ra.out = pl->tB;
          ra.prho = pc;
          ra.S = pl->S_all;
          ra.mask = pl->mask;
          ra.J = pl->J;
          ra.c_omega = pl->c_omega;
          ra.rho_omega = pl->rho_omega;
          TRY(q.kern("k234", [&] { return launch_k234(pl->ng, ra, pl->tw, q.s); }));
          c5.S = pl->S_all;
          c5.nS = pl->J;
        } else {
          RowArgs ra{};
          ra.in = pl->tA;
          ra.out = pl->tB;
          ra.prho = pc;
          TRY(q.row(RK_K2, ra));
          ColArgs c3{};
          c3.in = pl->tB;
          c3.out = pl->tA;
          TRY(q.col(CK_PSF, c3));
          TRY(enq_k4_allreduce(q));
          set_S(pl, c5);
        }
        c5.in = pl->tB;
        c5.src2 = pc + N;
        c5.out = pl->Ap + N;
        c5.rho_a = pc;
        c5.rho_out = pl->Ap;
        c5.alpha = alpha;
        c5.partials = pl->partials;
        c5.out_slot = SC_PAP_CHAT + it;
        c5.out_slot_rho = SC_PAP_RHO + it;
        c5.last_iter = (it == L - 1) ? 1 : 0;
        c5.fuse_k1 = (it < L - 1) ? 1 : 0;
        c5.iter = it;
        c5.r = pl->r + N;
        c5.rho_r = pl->r;
        c5.p = pc + N;
        c5.rho_p = pc;
        c5.dx = pl->dx + N;
        c5.rho_dx = pl->dx;
        c5.t1 = pl->tA;
        c5.xc = x + N;
        c5.x_rho = x;
        c5.bar_count = pl->kbar;
        c5.k5_rows = pl->k5_rows;
        c5.fold_sp = (it == L - 1) ? 1 : 0;
        c5.fpart = pl->kpart;
        if (pl->tmaps) {
          c5.tmap_r = pl->tmaps;
          c5.tmap_dx = pl->tmaps + 1;
          c5.tmap_p = pl->tmaps + 2;
        }
        TRY(q.col(CK_K5CG, c5));
      }
      sp_ready = L >= 1;
      continue;
    }
    // CG: L iterations of the normal operator + vector updates
    for (int it = 0; it < L; ++it) {
      TRY(enq_normal(q, alpha, pl->p, pl->Ap, true, it, L - 1));
      if (it < L - 1 && !pl->cg1) {  // r -= gamma Ap, <r, r> (dx is updated inside the next K1)
        VecArgs vr = q.vec();
        vr.r = pl->r;
        vr.Ap = pl->Ap;
        vr.iter = it;
        TRY(q.kern("r_update", [&] { return launch_r_update(pl->ng, vr, q.s); }));
        TRY(q.allreduce_scalar(SC_RR_CHAT + it + 1));
      }
    }
    // x_{n+1} = x_n + dx (+ gamma_{L-1} p_{L-1}, the step the next K1 would have taken)
    VecArgs vu = q.vec();
    vu.x = x;
    vu.dx = pl->dx;
    vu.p = pl->p;
    vu.iter = L;
    TRY(q.kern("newton_update", [&] { return launch_newton_update(pl->ng, vu, q.s); }));
  }
  if (img) {
    ColArgs ca{};
    ca.src = x + N;
    ca.out = pl->tA;
    if (!sp_ready) TRY(q.col(CK_IFFT_W, ca));
    RowArgs ra{};
    ra.in = pl->tA;
    ra.xrho = x;
    ra.rss = pl->rss_all;
    TRY(q.row(RK_RSS, ra));
    if (pl->p2p) {   // local RSS into the window, then one two-phase exchange (+ the residual history)
      float* wrss = reinterpret_cast<float*>(pl->xwin + kXWinHdr + 2 * pl->Q * sizeof(float2));
      TRY(q.kern("rss_sum", [&] { return launch_rss_sum(pl->ng, pl->rss_all, pl->J, wrss, q.s); }));
      TRY(enq_xchg_frame(q, K, pl->rss_sum));
      TRY(q.kern("image", [&] { return launch_image(pl->ng, pl->rho_omega, pl->rss_sum, 1, img, q.s); }));
    } else if (pl->multi) {
      TRY(q.kern("rss_sum", [&] { return launch_rss_sum(pl->ng, pl->rss_all, pl->J, pl->rss, q.s); }));
      TRY(q.allreduce_f(pl->rss, pl->rss_sum, pl->Q));
      TRY(q.kern("image", [&] { return launch_image(pl->ng, pl->rho_omega, pl->rss_sum, 1, img, q.s); }));
    } else {
      TRY(q.kern("image", [&] { return launch_image(pl->ng, pl->rho_omega, pl->rss_all, pl->J, img, q.s); }));
    }
  } else if (pl->p2p) {
    TRY(enq_xchg_frame(q, K, nullptr));   // the residual history is a sum over all ranks' coils
  }
  return NLINV_OK;
}

}  // namespace

// ------------------------------------------------------------------ operator entry points
extern "C" nlinv_status nlinv_set_point(nlinv_plan pl, const nlinv_c32* x, void* stream) {
  if (!pl || !x) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  Enq q{pl, (cudaStream_t)stream};
  nlinv_status st = enq_set_point(q, (const float2*)x, nullptr);
  pl->launches += q.kernels;
  if (st == NLINV_OK) pl->point_set = true;
  return st;
}

extern "C" nlinv_status nlinv_apply_forward(nlinv_plan pl, const nlinv_c32* x, nlinv_c32* y, void* stream) {
  if (!pl || !x || !y) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  Enq q{pl, (cudaStream_t)stream};
  nlinv_status st = enq_set_point(q, (const float2*)x, pl->tB);
  if (st == NLINV_OK) {
    pl->point_set = true;
    ColArgs ca{};
    ca.in = pl->tB;
    ca.out = (float2*)y;
    st = q.col(CK_FWDP, ca);
  }
  pl->launches += q.kernels;
  return st;
}

extern "C" nlinv_status nlinv_apply_derivative(nlinv_plan pl, const nlinv_c32* dx, nlinv_c32* dy, void* stream) {
  if (!pl || !dx || !dy) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (!pl->point_set) return fail(pl, NLINV_ERR_STATE, "derivative before set_point");
  Enq q{pl, (cudaStream_t)stream};
  nlinv_status st = enq_derivative_head(q, (const float2*)dx, false, 0);
  if (st == NLINV_OK) {
    ColArgs ca{};
    ca.in = pl->tB;
    ca.out = (float2*)dy;
    st = q.col(CK_FWDP, ca);
  }
  pl->launches += q.kernels;
  return st;
}

extern "C" nlinv_status nlinv_apply_adjoint(nlinv_plan pl, const nlinv_c32* dy, nlinv_c32* dx, void* stream) {
  if (!pl || !dy || !dx) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (!pl->point_set) return fail(pl, NLINV_ERR_STATE, "adjoint before set_point");
  if (pl->p2p && pl->xp.G == 0) return fail(pl, NLINV_ERR_STATE, "peer-memory plan used before nlinv_plan_connect");
  Enq q{pl, (cudaStream_t)stream};
  auto body = [&]() -> nlinv_status {
    ColArgs ca{};
    ca.in = (const float2*)dy;
    ca.out = pl->tA;
    TRY(q.col(CK_ADJ1, ca));
    TRY(enq_k4_allreduce(q));
    ColArgs cb{};
    cb.in = pl->tB;
    cb.out = (float2*)dx + pl->N;
    set_S(pl, cb);
    cb.rho_out = (float2*)dx;
    TRY(q.col(CK_FFT_W_ADJ, cb));
    return NLINV_OK;
  };
  nlinv_status st = body();
  pl->launches += q.kernels;
  return st;
}

extern "C" nlinv_status nlinv_apply_normal(nlinv_plan pl, float alpha, const nlinv_c32* dx, nlinv_c32* out,
                                           void* stream) {
  if (!pl || !dx || !out) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (dx == out) return fail(pl, NLINV_ERR_ARG, "dx and out must not overlap");
  if (!pl->point_set) return fail(pl, NLINV_ERR_STATE, "normal before set_point");
  if (pl->p2p && pl->xp.G == 0) return fail(pl, NLINV_ERR_STATE, "peer-memory plan used before nlinv_plan_connect");
  Enq q{pl, (cudaStream_t)stream};
  nlinv_status st = enq_normal(q, alpha, (const float2*)dx, (float2*)out, false, 0);
  pl->launches += q.kernels;
  return st;
}

extern "C" nlinv_status nlinv_debug_fft2d(nlinv_plan pl, const nlinv_c32* in, nlinv_c32* out, int batch, int inverse,
                                          void* stream) {
  if (!pl || !in || !out) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (batch < 1) return fail(pl, NLINV_ERR_ARG, "batch < 1");
  cudaError_t e = launch_fft2d(pl->ng, (const float2*)in, (float2*)out, batch, inverse, pl->tw, nullptr,
                               (cudaStream_t)stream);
  pl->launches += 2;
  if (e != cudaSuccess) return fail(pl, NLINV_ERR_CUDA, std::string("fft2d: ") + cudaGetErrorString(e));
  return NLINV_OK;
}

// ------------------------------------------------------------------ reconstruct
static nlinv_status reconstruct_on(nlinv_plan pl, const nlinv_c32* frame, const nlinv_c32* prior, int newton_steps,
                                   int cg_iters, nlinv_c32* x_out, nlinv_c32* image_out, cudaStream_t s);

extern "C" nlinv_status nlinv_reconstruct(nlinv_plan pl, const nlinv_c32* frame, const nlinv_c32* prior,
                                          int newton_steps, int cg_iters, nlinv_c32* x_out, nlinv_c32* image_out,
                                          void* stream) {
  if (!pl || !frame || !x_out) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (newton_steps < 0 || newton_steps > kMaxNewton) return fail(pl, NLINV_ERR_SIZE, "newton_steps out of range");
  if (cg_iters < 1 || cg_iters > kMaxCG) return fail(pl, NLINV_ERR_SIZE, "cg_iters out of range");
  if (pl->p2p && pl->xp.G == 0) return fail(pl, NLINV_ERR_STATE, "peer-memory plan used before nlinv_plan_connect");
  cudaStream_t us = (cudaStream_t)stream;
  // A CUDA graph cannot be captured on the legacy default stream: callers on it (e.g. torch's
  // default stream) get the frame's graph on a plan-owned stream fenced by events on both sides,
  // so the call stays stream-ordered with respect to `stream`.
  const bool graphs = !pl->prof && (std::getenv("NLINV_NO_GRAPH") == nullptr);
  if (us == nullptr && graphs) {
    if (!pl->gstream) {
      CU(cudaStreamCreateWithFlags(&pl->gstream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&pl->gev_in, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&pl->gev_out, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(pl->gev_in, us));
    CU(cudaStreamWaitEvent(pl->gstream, pl->gev_in, 0));
    nlinv_status st = reconstruct_on(pl, frame, prior, newton_steps, cg_iters, x_out, image_out, pl->gstream);
    CU(cudaEventRecord(pl->gev_out, pl->gstream));
    CU(cudaStreamWaitEvent(us, pl->gev_out, 0));
    return st;
  }
  return reconstruct_on(pl, frame, prior, newton_steps, cg_iters, x_out, image_out, us);
}

static nlinv_status reconstruct_on(nlinv_plan pl, const nlinv_c32* frame, const nlinv_c32* prior, int newton_steps,
                                   int cg_iters, nlinv_c32* x_out, nlinv_c32* image_out, cudaStream_t s) {
  pl->last_stream = s;
  pl->last_K = newton_steps;
  pl->last_L = cg_iters;
  GraphKey key;
  key.frame = frame;
  key.prior = prior;
  key.xout = x_out;
  key.img = image_out;
  key.K = newton_steps;
  key.L = cg_iters;
  key.stream = s;
  key.pw = pl->pw_active;
  const bool use_graph = (s != nullptr) && !pl->prof && (std::getenv("NLINV_NO_GRAPH") == nullptr);
  if (use_graph && pl->gexec && pl->gkey == key) {
    CU(cudaGraphLaunch(pl->gexec, s));
    pl->launches += pl->gkernels;
    pl->point_set = true;
    return NLINV_OK;
  }
  Enq q{pl, s};
  if (!use_graph) {
    nlinv_status st = enq_reconstruct(q, (const float2*)frame, (const float2*)prior, newton_steps, cg_iters,
                                      (float2*)x_out, (float2*)image_out);
    pl->launches += q.kernels;
    pl->point_set = true;
    return st;
  }
  if (pl->gexec) {
    cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
  }
  CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  nlinv_status st = enq_reconstruct(q, (const float2*)frame, (const float2*)prior, newton_steps, cg_iters,
                                    (float2*)x_out, (float2*)image_out);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &graph);
  if (st != NLINV_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(pl, NLINV_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&pl->gexec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    pl->gexec = nullptr;
    return fail(pl, NLINV_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  }
  pl->gkey = key;
  pl->gkernels = q.kernels;
  CU(cudaGraphLaunch(pl->gexec, s));
  pl->launches += pl->gkernels;
  pl->point_set = true;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_reconstruct_host(nlinv_plan pl, const nlinv_c32* frame, const nlinv_c32* prior,
                                               int newton_steps, int cg_iters, nlinv_c32* x_out,
                                               nlinv_c32* image_out, void* stream) {
  if (!pl || !frame) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  const size_t N = pl->N, tot = N * (1 + pl->J);
  cudaStream_t s = (cudaStream_t)stream;
  if (!pl->h_frame) {
    CU(cudaMalloc((void**)&pl->h_frame, sizeof(float2) * N * pl->J));
    CU(cudaMalloc((void**)&pl->h_x, sizeof(float2) * tot));
    CU(cudaMalloc((void**)&pl->h_img, sizeof(float2) * pl->Q));
  }
  CU(cudaMemcpyAsync(pl->h_frame, frame, sizeof(float2) * N * pl->J, cudaMemcpyHostToDevice, s));
  if (prior) CU(cudaMemcpyAsync(pl->h_x, prior, sizeof(float2) * tot, cudaMemcpyHostToDevice, s));
  nlinv_status st = nlinv_reconstruct(pl, (const nlinv_c32*)pl->h_frame, prior ? (const nlinv_c32*)pl->h_x : nullptr,
                                      newton_steps, cg_iters, (nlinv_c32*)pl->h_x,
                                      image_out ? (nlinv_c32*)pl->h_img : nullptr, stream);
  if (st != NLINV_OK) return st;
  if (x_out) CU(cudaMemcpyAsync(x_out, pl->h_x, sizeof(float2) * tot, cudaMemcpyDeviceToHost, s));
  if (image_out) CU(cudaMemcpyAsync(image_out, pl->h_img, sizeof(float2) * pl->Q, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_stats(nlinv_plan pl, nlinv_stats* out) {
  if (!pl || !out) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  CU(cudaStreamSynchronize(pl->last_stream));
  std::vector<double> sc(SC_TOTAL);
  CU(cudaMemcpy(sc.data(), pl->scal, sizeof(double) * SC_TOTAL, cudaMemcpyDeviceToHost));
  std::memset(out, 0, sizeof(*out));
  out->newton_done = pl->last_K;
  for (int k = 0; k < pl->last_K && k < 64; ++k) out->residual[k] = std::sqrt(sc[SC_RES + k]);
  // breakdown: <r,r> exactly zero inside the last solve (A9)
  for (int i = 0; i < pl->last_L; ++i)
    if (sc[SC_RR_RHO + i] + sc[SC_RR_CHAT + i] == 0.0) out->cg_breakdown = 1;
  for (int k = 1; k < pl->last_K && k < 64; ++k)
    if (out->residual[k] > 10.0 * out->residual[0]) out->diverged = 1;
  return NLINV_OK;
}

// ------------------------------------------------------------------ streaming (real-time) entry
extern "C" nlinv_status nlinv_stream_reset(nlinv_plan pl) {
  if (!pl) return fail(pl, NLINV_ERR_ARG, "NULL plan");
  pl->stream_started = false;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_stream_frame(nlinv_plan pl, const nlinv_c32* frame_host, const uint8_t* mask_host,
                                           int newton_steps, int cg_iters, nlinv_c32* image_host, void* stream) {
  if (!pl || !frame_host) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  const size_t N = pl->N, tot = N * (1 + pl->J);
  cudaStream_t s = (cudaStream_t)stream;
  if (!pl->h_frame) {
    CU(cudaMalloc((void**)&pl->h_frame, sizeof(float2) * N * pl->J));
    CU(cudaMalloc((void**)&pl->h_x, sizeof(float2) * tot));
    CU(cudaMalloc((void**)&pl->h_img, sizeof(float2) * pl->Q));
  }
  CU(cudaMemcpyAsync(pl->h_frame, frame_host, sizeof(float2) * N * pl->J, cudaMemcpyHostToDevice, s));
  if (mask_host) {
    CU(cudaMemcpyAsync(pl->mask, mask_host, N, cudaMemcpyHostToDevice, s));
    pl->pw_active = nullptr;   // a binary P_k from the host replaces any KB weights
    pl->mnnz_host = -1;
  }
  nlinv_status st = nlinv_reconstruct(pl, (const nlinv_c32*)pl->h_frame,
                                      pl->stream_started ? (const nlinv_c32*)pl->h_x : nullptr, newton_steps,
                                      cg_iters, (nlinv_c32*)pl->h_x, image_host ? (nlinv_c32*)pl->h_img : nullptr,
                                      stream);
  if (st != NLINV_OK) return st;
  pl->stream_started = true;
  if (image_host) CU(cudaMemcpyAsync(image_host, pl->h_img, sizeof(float2) * pl->Q, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return NLINV_OK;
}

// ------------------------------------------------------------------ per-kernel profiling
extern "C" nlinv_status nlinv_plan_set_profiling(nlinv_plan pl, int on) {
  if (!pl) return fail(pl, NLINV_ERR_ARG, "NULL plan");
  pl->prof = on != 0;
  pl->prof_rec.clear();
  pl->ev_used = 0;
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_profile_json(nlinv_plan pl, char* buf, size_t len) {
  if (!pl || !buf || len == 0) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  CU(cudaDeviceSynchronize());
  std::vector<std::string> names;
  std::vector<double> ms;
  std::vector<long long> cnt;
  for (const auto& r : pl->prof_rec) {
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, r.e0, r.e1));
    size_t k = 0;
    while (k < names.size() && names[k] != r.name) ++k;
    if (k == names.size()) {
      names.push_back(r.name);
      ms.push_back(0.0);
      cnt.push_back(0);
    }
    ms[k] += t;
    cnt[k] += 1;
  }
  std::string out = "{";
  for (size_t k = 0; k < names.size(); ++k) {
    char tmp[160];
    std::snprintf(tmp, sizeof(tmp), "%s\"%s\": [%lld, %.6f]", k ? ", " : "", names[k].c_str(), cnt[k], ms[k]);
    out += tmp;
  }
  out += "}";
  pl->prof_rec.clear();
  pl->ev_used = 0;
  if (out.size() + 1 > len) return fail(pl, NLINV_ERR_SIZE, "profile buffer too small");
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return NLINV_OK;
}

// ------------------------------------------------------------------ debug CTA timelines (-DNLV_TRACE)
extern "C" nlinv_status nlinv_plan_trace(nlinv_plan pl, int col_mode, unsigned long long* out, int cap) {
  if (!pl) return fail(pl, NLINV_ERR_ARG, "NULL plan");
  if (col_mode >= 0) {
    if (!pl->trace) CU(cudaMalloc((void**)&pl->trace, sizeof(unsigned long long) * 8 * 8192));
    CU(cudaMemset(pl->trace, 0, sizeof(unsigned long long) * 8 * 8192));
    pl->trace_mode = col_mode;
    return NLINV_OK;
  }
  if (!pl->trace || !out) return fail(pl, NLINV_ERR_STATE, "trace not enabled");
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(out, pl->trace, sizeof(unsigned long long) * (cap < 8 * 8192 ? cap : 8 * 8192), cudaMemcpyDeviceToHost));
  pl->trace_mode = -1;
  return NLINV_OK;
}

// ------------------------------------------------------------------ P_k index list and compact ingest
static nlinv_status ensure_index_buffers(nlinv_plan pl) {
  if (!pl->midx) {
    CU(cudaMalloc((void**)&pl->midx, sizeof(int) * pl->N));
    CU(cudaMalloc((void**)&pl->mcount, sizeof(int) * mask_count_blocks((int)pl->N)));
    CU(cudaMalloc((void**)&pl->mnnz, sizeof(int)));
  }
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_mask_indices(nlinv_plan pl, int* idx_host, int cap, int* nnz_host, void* stream) {
  if (!pl || !nnz_host) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  nlinv_status st = ensure_index_buffers(pl);
  if (st != NLINV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  CU(launch_mask_compact(pl->mask, (int)pl->N, pl->mcount, pl->midx, pl->mnnz, s));
  pl->launches += 2;
  int nnz = 0;
  CU(cudaMemcpyAsync(&nnz, pl->mnnz, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *nnz_host = nnz;
  pl->mnnz_host = nnz;
  if (idx_host) {
    if (cap < nnz) return fail(pl, NLINV_ERR_SIZE, "idx buffer smaller than nnz");
    CU(cudaMemcpy(idx_host, pl->midx, sizeof(int) * nnz, cudaMemcpyDeviceToHost));
  }
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_stream_frame_compact(nlinv_plan pl, const nlinv_c32* samples_host, int nnz,
                                                   const uint8_t* mask_host, int newton_steps, int cg_iters,
                                                   nlinv_c32* image_host, void* stream) {
  if (!pl || !samples_host || nnz < 0 || (size_t)nnz > pl->N) return fail(pl, NLINV_ERR_ARG, "bad argument");
  const size_t N = pl->N, tot = N * (1 + pl->J);
  cudaStream_t s = (cudaStream_t)stream;
  nlinv_status st = ensure_index_buffers(pl);
  if (st != NLINV_OK) return st;
  if (!pl->h_frame) {
    CU(cudaMalloc((void**)&pl->h_frame, sizeof(float2) * N * pl->J));
    CU(cudaMemset(pl->h_frame, 0, sizeof(float2) * N * pl->J));
    CU(cudaMalloc((void**)&pl->h_x, sizeof(float2) * tot));
    CU(cudaMalloc((void**)&pl->h_img, sizeof(float2) * pl->Q));
  }
  if (!pl->h_samples) CU(cudaMalloc((void**)&pl->h_samples, sizeof(float2) * N * pl->J));
  if (mask_host) {
    long long cnt = 0;
    for (size_t i = 0; i < N; ++i) cnt += mask_host[i] ? 1 : 0;
    CU(cudaMemcpyAsync(pl->mask, mask_host, N, cudaMemcpyHostToDevice, s));
    pl->pw_active = nullptr;   // a binary P_k from the host replaces any KB weights
    CU(launch_mask_compact(pl->mask, (int)N, pl->mcount, pl->midx, pl->mnnz, s));
    pl->launches += 2;
    pl->mnnz_host = cnt;
  } else if (pl->mnnz_host < 0) {
    int cnt = 0;
    st = nlinv_mask_indices(pl, nullptr, 0, &cnt, stream);
    if (st != NLINV_OK) return st;
    pl->mnnz_host = cnt;
  }
  if ((long long)nnz != pl->mnnz_host) return fail(pl, NLINV_ERR_SIZE, "nnz differs from the sampled-cell count of P_k");
  CU(cudaMemcpyAsync(pl->h_samples, samples_host, sizeof(float2) * (size_t)nnz * pl->J, cudaMemcpyHostToDevice, s));
  CU(launch_scatter_samples(pl->h_samples, pl->midx, pl->mnnz, nnz, pl->J, N, pl->h_frame, s));
  pl->launches += 1;
  st = nlinv_reconstruct(pl, (const nlinv_c32*)pl->h_frame, pl->stream_started ? (const nlinv_c32*)pl->h_x : nullptr,
                         newton_steps, cg_iters, (nlinv_c32*)pl->h_x, image_host ? (nlinv_c32*)pl->h_img : nullptr,
                         stream);
  if (st != NLINV_OK) return st;
  pl->stream_started = true;
  if (image_host) CU(cudaMemcpyAsync(image_host, pl->h_img, sizeof(float2) * pl->Q, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_stream_frame_radial(nlinv_plan pl, const nlinv_c32* raw_host, int frame, int newton_steps,
                                                  int cg_iters, nlinv_c32* image_host, void* stream) {
  if (!pl || !raw_host || frame < 0) return fail(pl, NLINV_ERR_ARG, "bad argument");
  if (pl->traj_turns == 0) return fail(pl, NLINV_ERR_STATE, "nlinv_stream_frame_radial before nlinv_plan_set_trajectory");
  const size_t N = pl->N, tot = N * (1 + pl->J);
  const size_t nraw = (size_t)pl->traj_spokes * pl->ng;
  cudaStream_t s = (cudaStream_t)stream;
  if (!pl->h_frame) {
    CU(cudaMalloc((void**)&pl->h_frame, sizeof(float2) * N * pl->J));
    CU(cudaMemset(pl->h_frame, 0, sizeof(float2) * N * pl->J));
    CU(cudaMalloc((void**)&pl->h_x, sizeof(float2) * tot));
    CU(cudaMalloc((void**)&pl->h_img, sizeof(float2) * pl->Q));
  }
  if (!pl->h_raw) CU(cudaMalloc((void**)&pl->h_raw, sizeof(float2) * nraw * pl->J));
  CU(cudaMemcpyAsync(pl->h_raw, raw_host, sizeof(float2) * nraw * pl->J, cudaMemcpyHostToDevice, s));
  nlinv_status st = nlinv_grid_radial(pl, frame, (const nlinv_c32*)pl->h_raw, (nlinv_c32*)pl->h_frame, stream);
  if (st != NLINV_OK) return st;
  st = nlinv_reconstruct(pl, (const nlinv_c32*)pl->h_frame, pl->stream_started ? (const nlinv_c32*)pl->h_x : nullptr,
                         newton_steps, cg_iters, (nlinv_c32*)pl->h_x, image_host ? (nlinv_c32*)pl->h_img : nullptr,
                         stream);
  if (st != NLINV_OK) return st;
  pl->stream_started = true;
  if (image_host) CU(cudaMemcpyAsync(image_host, pl->h_img, sizeof(float2) * pl->Q, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return NLINV_OK;
}

// debug: co-resident clusters of the cluster-fused K2-K3-K4 kernel at grid size ng (< 0: not built)
extern "C" int nlinv_debug_k234_clusters(int ng) { return k234_max_clusters(ng); }

// ------------------------------------------------------------------ peer-memory exchange
extern "C" nlinv_status nlinv_plan_exchange_handle(nlinv_plan pl, unsigned char handle[64]) {
  if (!pl || !handle) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (!pl->p2p) return fail(pl, NLINV_ERR_STATE, "not a peer-memory plan (world == 1 or NCCL transport)");
  cudaIpcMemHandle_t h;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
  CU(cudaIpcGetMemHandle(&h, pl->xwin));
  std::memcpy(handle, &h, 64);
  return NLINV_OK;
}

static nlinv_status connect_done(nlinv_plan pl) {
  pl->xp.G = pl->world;
  pl->xp.rank = pl->rank;
  if (!pl->xp_dev) CU(cudaMalloc((void**)&pl->xp_dev, sizeof(XPeers)));
  CU(cudaMemcpy(pl->xp_dev, &pl->xp, sizeof(XPeers), cudaMemcpyHostToDevice));
  if (pl->gexec) {   // a graph captured before the peers were known is stale
    cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
  }
  return NLINV_OK;
}

extern "C" nlinv_status nlinv_plan_connect(nlinv_plan pl, const unsigned char* handles) {
  if (!pl || !handles) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (!pl->p2p) return fail(pl, NLINV_ERR_STATE, "not a peer-memory plan (world == 1 or NCCL transport)");
  if (pl->xp.G) return fail(pl, NLINV_ERR_STATE, "already connected");
  for (int r = 0; r < pl->world; ++r) {
    if (r == pl->rank) {
      pl->xp.win[r] = pl->xwin;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * r, 64);
    void* ptr = nullptr;
    CU(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    pl->ipc_open.push_back(ptr);
    pl->xp.win[r] = static_cast<char*>(ptr);
  }
  return connect_done(pl);
}

extern "C" nlinv_status nlinv_plan_connect_local(nlinv_plan pl, const nlinv_plan* plans) {
  if (!pl || !plans) return fail(pl, NLINV_ERR_ARG, "NULL argument");
  if (!pl->p2p) return fail(pl, NLINV_ERR_STATE, "not a peer-memory plan (world == 1 or NCCL transport)");
  if (pl->xp.G) return fail(pl, NLINV_ERR_STATE, "already connected");
  for (int r = 0; r < pl->world; ++r) {
    const nlinv_plan o = plans[r];
    if (!o || !o->p2p || o->rank != r || o->world != pl->world || o->ng != pl->ng)
      return fail(pl, NLINV_ERR_ARG, "plans[] must be this job's peer-memory plans in rank order");
    if (o->device != pl->device) {   // another GPU of this process: direct peer access over NVLink
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, pl->device, o->device));
      if (!can) return fail(pl, NLINV_ERR_CUDA, "no peer access between the plans' devices");
      cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CU(e);
      cudaGetLastError();
    }
    pl->xp.win[r] = o->xwin;
  }
  return connect_done(pl);
}

extern "C" nlinv_status nlinv_debug_axpy(float a, const float* x, float* y, long long n, void* stream) {
  nlinv_plan pl = nullptr;
  if (!x || !y || n < 0 || n % 4) return fail(pl, NLINV_ERR_ARG, "axpy: NULL pointer or n not a multiple of 4");
  CU(launch_axpy(a, x, y, n, (cudaStream_t)stream));
  return NLINV_OK;
}
