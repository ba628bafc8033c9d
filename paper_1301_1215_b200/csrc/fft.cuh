// Register/shared-memory mixed-radix FFT building blocks for sm_100a.
//
// The paper's operators are built from 2D DFTs applied per coil channel ("a number of
// Fourier transform calculations applied separately to each channel") and
// the FFT is "the most time-consuming operation". The paper called batched cuFFT;
// here a length-L transform is a short sequence of Stockham autosort passes whose
// butterflies live in registers, with one shared-memory exchange between passes.
//
//   L = R_0 * R_1 * ... * R_{P-1},  T threads per transform, E = L / T values per thread.
//   Pass p (stride Ns = R_0 ... R_{p-1}): thread t handles butterflies j = t + T*m,
//   m in [0, E/R_p); butterfly j reads x[j + r L/R_p], multiplies by w_{Ns R_p}^{(j mod Ns) r},
//   runs a radix-R_p DFT and writes x[(j/Ns) Ns R_p + (j mod Ns) + r Ns].
//
// The input pattern of pass 0 and the output pattern of the last pass are both
// "index = t + T*m + r*L/R", so global loads/stores of consecutive t are contiguous, and a
// schedule with R_0 == R_{P-1} lets an inverse transform feed a forward one in registers.
// Twiddles come from a per-CTA shared table computed in fp64 on the host (no __sinf).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nlv {

// ------------------------------------------------------------------ complex helpers
// sm_100a has packed two-lane fp32 instructions (FADD2 / FMUL2 / FFMA2: one instruction, both halves of a
// register pair, each lane IEEE round-to-nearest like FADD / FMUL / FFMA): a complex add is one
// instruction instead of two. ptxas folds lane broadcasts and the re/im swap into operand modifiers
// (.F32 / .LO_HI), so a complex multiply is two or three. Measured lane throughput equals the scalar
// pipe's (tools/probe_f32x2), so the gain is issue slots, which bound these FFT passes.
#ifndef NLV_SCALAR_FP
__device__ __forceinline__ unsigned long long pk2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}

__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}

// lane-wise a * b + c, one rounding per lane
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  return up2(r);
}
#else   // scalar reference of the same lane-wise operations (A/B builds)
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
#endif
__device__ __forceinline__ float2 swap2(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 bcast2(float s) { return make_float2(s, s); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
// a * b = b.x a + b.y (-a.y, a.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return fma2(swap2(a), make_float2(-b.y, b.y), mul2(a, bcast2(b.x)));
}
// conj(a) * b = a.x b + a.y (b.y, -b.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return fma2(swap2(b), make_float2(a.y, -a.y), mul2(b, bcast2(a.x)));
}
// scalar on purpose: the packed form (FMUL2 with a broadcast scalar) gave wrong results in the
// ng = 16 / 48 adjoint passes (measured, tools/dbg_adj.py); the scalar pair costs one extra FMUL
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cneg_if(float2 a, bool neg) { return neg ? make_float2(-a.x, -a.y) : a; }
// a * (DIR * i)
template <int DIR>
__device__ __forceinline__ float2 mul_dir_i(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
// a + DIR i b and a - DIR i b, each one FFMA2 (b swapped, lane signs as an immediate pair)
template <int DIR>
__device__ __forceinline__ float2 cadd_i(float2 a, float2 b) {
  return fma2(swap2(b), DIR < 0 ? make_float2(1.f, -1.f) : make_float2(-1.f, 1.f), a);
}
template <int DIR>
__device__ __forceinline__ float2 csub_i(float2 a, float2 b) {
  return fma2(swap2(b), DIR < 0 ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f), a);
}
// e^{DIR 2 pi i m / R} for compile-time-foldable m, R with 48 % R == 0 (R in {2,3,4,6,8,12,16})
template <int DIR>
__device__ __forceinline__ float2 unit_root48(int k48) {
  constexpr float c[48] = {
      1.000000000e+00f, 9.914448614e-01f, 9.659258263e-01f, 9.238795325e-01f, 8.660254038e-01f, 7.933533403e-01f,
      7.071067812e-01f, 6.087614290e-01f, 5.000000000e-01f, 3.826834324e-01f, 2.588190451e-01f, 1.305261922e-01f,
      0.0f, -1.305261922e-01f, -2.588190451e-01f, -3.826834324e-01f, -5.000000000e-01f, -6.087614290e-01f,
      -7.071067812e-01f, -7.933533403e-01f, -8.660254038e-01f, -9.238795325e-01f, -9.659258263e-01f, -9.914448614e-01f,
      -1.000000000e+00f, -9.914448614e-01f, -9.659258263e-01f, -9.238795325e-01f, -8.660254038e-01f, -7.933533403e-01f,
      -7.071067812e-01f, -6.087614290e-01f, -5.000000000e-01f, -3.826834324e-01f, -2.588190451e-01f, -1.305261922e-01f,
      0.0f, 1.305261922e-01f, 2.588190451e-01f, 3.826834324e-01f, 5.000000000e-01f, 6.087614290e-01f,
      7.071067812e-01f, 7.933533403e-01f, 8.660254038e-01f, 9.238795325e-01f, 9.659258263e-01f, 9.914448614e-01f};
  const int ks = (k48 + 36) % 48;  // sin(theta) = cos(theta - pi/2)
  return make_float2(c[k48], DIR * c[ks]);
}

// ------------------------------------------------------------------ small DFTs (in registers)
// X_k = sum_n a_n e^{DIR 2 pi i n k / R}; natural order in and out.
template <int R, int DIR>
struct DFT;

template <int DIR>
struct DFT<1, DIR> {
  __device__ __forceinline__ static void run(float2*) {}
};

template <int DIR>
struct DFT<2, DIR> {
  __device__ __forceinline__ static void run(float2* a) {
    float2 t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  }
};

template <int DIR>
struct DFT<3, DIR> {
  __device__ __forceinline__ static void run(float2* a) {
    const float s = DIR * 0.866025403784438647f;
    float2 t1 = cadd(a[1], a[2]);
    float2 t2 = csub(a[1], a[2]);
    float2 m = fma2(bcast2(-0.5f), t1, a[0]);
    a[0] = cadd(a[0], t1);
    a[1] = fma2(swap2(t2), make_float2(-s, s), m);   // m + i s t2
    a[2] = fma2(swap2(t2), make_float2(s, -s), m);   // m - i s t2
  }
};

template <int DIR>
struct DFT<4, DIR> {
  __device__ __forceinline__ static void run(float2* a) {
    float2 t0 = cadd(a[0], a[2]);
    float2 t1 = csub(a[0], a[2]);
    float2 t2 = cadd(a[1], a[3]);
    float2 d3 = csub(a[1], a[3]);
    a[0] = cadd(t0, t2);
    a[2] = csub(t0, t2);
    a[1] = cadd_i<DIR>(t1, d3);
    a[3] = csub_i<DIR>(t1, d3);
  }
};

// a * e^{DIR 2 pi i k48 / 48} for a compile-time k48: quarter turns are exact sign/swap moves
// (a multiply by the literal 0 cannot be folded under IEEE rules, so cmul would waste 4 FP ops),
// eighth turns use (x -+ y) sqrt(1/2) (2 FADD + 2 FMUL), the rest a full complex multiply.
template <int DIR>
__device__ __forceinline__ float2 mul_root48(float2 a, int k48) {
  const int k = ((k48 % 48) + 48) % 48;
  if (k == 0) return a;
  if (k == 24) return make_float2(-a.x, -a.y);
  if (k == 12) return mul_dir_i<DIR>(a);                       // e^{DIR i pi/2} = DIR i
  if (k == 36) return mul_dir_i<-DIR>(a);
  constexpr float h = 0.707106781186547524f;
  // eighth turns: h (a + swap(a) (s0, s1)) with the lane signs of each case (one FFMA2 + one FMUL2)
  if (k == 6) return DIR < 0 ? cscale(fma2(swap2(a), make_float2(1.f, -1.f), a), h) : cscale(fma2(swap2(a), make_float2(-1.f, 1.f), a), h);
  if (k == 18) return DIR < 0 ? cscale(fma2(swap2(a), make_float2(1.f, -1.f), make_float2(-a.x, -a.y)), h)
                              : cscale(fma2(swap2(a), make_float2(-1.f, 1.f), make_float2(-a.x, -a.y)), h);
  if (k == 30) return DIR < 0 ? cscale(fma2(swap2(a), make_float2(-1.f, 1.f), make_float2(-a.x, -a.y)), h)
                              : cscale(fma2(swap2(a), make_float2(1.f, -1.f), make_float2(-a.x, -a.y)), h);
  if (k == 42) return DIR < 0 ? cscale(fma2(swap2(a), make_float2(-1.f, 1.f), a), h) : cscale(fma2(swap2(a), make_float2(1.f, -1.f), a), h);
  return cmul(a, unit_root48<DIR>(k));
}

// Cooley-Tukey split R = R1*R2 entirely in registers: n = R2 n1 + n2, k = k1 + R1 k2.
template <int R1, int R2, int DIR>
__device__ __forceinline__ void dft_split(float2* a) {
  constexpr int R = R1 * R2;
  float2 b[R];
#pragma unroll
  for (int n2 = 0; n2 < R2; ++n2) {
    float2 t[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) t[n1] = a[R2 * n1 + n2];
    DFT<R1, DIR>::run(t);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int m = (n2 * k1) % R;
      b[n2 * R1 + k1] = mul_root48<DIR>(t[k1], m * (48 / R));
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    float2 t[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) t[n2] = b[n2 * R1 + k1];
    DFT<R2, DIR>::run(t);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) a[k1 + R1 * k2] = t[k2];
  }
}

template <int DIR>
struct DFT<6, DIR> {
  __device__ __forceinline__ static void run(float2* a) { dft_split<2, 3, DIR>(a); }
};
template <int DIR>
struct DFT<8, DIR> {
  __device__ __forceinline__ static void run(float2* a) { dft_split<2, 4, DIR>(a); }
};
template <int DIR>
struct DFT<12, DIR> {
  __device__ __forceinline__ static void run(float2* a) { dft_split<4, 3, DIR>(a); }
};
template <int DIR>
struct DFT<16, DIR> {
  __device__ __forceinline__ static void run(float2* a) { dft_split<4, 4, DIR>(a); }
};

// ------------------------------------------------------------------ zero-aware DFTs (pass 0 pruning)
// Pass 0 of a transform whose input is known zero on fixed register slots (the Omega-pruned half
// images: rows / columns outside Omega are structurally zero) skips the additions with those zeros:
// bit n of ZM marks input n of the small DFT as zero (compile time). Adding a literal 0 cannot be
// folded by the compiler under IEEE rules (-0 + 0 = +0), so this is done by hand.
template <bool ZA, bool ZB>
__device__ __forceinline__ float2 zadd(float2 a, float2 b) {
  if constexpr (ZA && ZB) return make_float2(0.f, 0.f);
  else if constexpr (ZA) return b;
  else if constexpr (ZB) return a;
  else return cadd(a, b);
}
template <bool ZA, bool ZB>
__device__ __forceinline__ float2 zsub(float2 a, float2 b) {
  if constexpr (ZA && ZB) return make_float2(0.f, 0.f);
  else if constexpr (ZA) return make_float2(-b.x, -b.y);
  else if constexpr (ZB) return a;
  else return csub(a, b);
}

template <int R, int DIR, unsigned ZM>
struct DFTZ {   // generic fallback: no pruning unless every input is zero
  __device__ __forceinline__ static void run(float2* a) {
    if constexpr (ZM != (1u << R) - 1u) DFT<R, DIR>::run(a);
  }
};
template <int DIR, unsigned ZM>
struct DFTZ<2, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) {
    constexpr bool z0 = ZM & 1u, z1 = (ZM >> 1) & 1u;
    const float2 t = a[0];
    a[0] = zadd<z0, z1>(t, a[1]);
    a[1] = zsub<z0, z1>(t, a[1]);
  }
};
template <int DIR, unsigned ZM>
struct DFTZ<4, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) {
    constexpr bool z0 = ZM & 1u, z1 = (ZM >> 1) & 1u, z2 = (ZM >> 2) & 1u, z3 = (ZM >> 3) & 1u;
    constexpr bool zt0 = z0 && z2, zt2 = z1 && z3;
    const float2 t0 = zadd<z0, z2>(a[0], a[2]);
    const float2 t1 = zsub<z0, z2>(a[0], a[2]);
    const float2 t2 = zadd<z1, z3>(a[1], a[3]);
    const float2 d3 = zsub<z1, z3>(a[1], a[3]);
    a[0] = zadd<zt0, zt2>(t0, t2);
    a[2] = zsub<zt0, zt2>(t0, t2);
    if constexpr (zt0 && zt2) {
      a[1] = a[3] = make_float2(0.f, 0.f);
    } else if constexpr (zt2) {
      a[1] = a[3] = t1;
    } else if constexpr (zt0) {
      a[1] = mul_dir_i<DIR>(d3);
      a[3] = mul_dir_i<-DIR>(d3);
    } else {
      a[1] = cadd_i<DIR>(t1, d3);
      a[3] = csub_i<DIR>(t1, d3);
    }
  }
};
// group mask of the n2-th stride-R2 subsequence (n = R2 n1 + n2) of a length-R1*R2 input
template <int R1, int R2>
__host__ __device__ constexpr unsigned split_group_mask(unsigned zm, int n2) {
  unsigned g = 0;
  for (int n1 = 0; n1 < R1; ++n1) g |= ((zm >> (R2 * n1 + n2)) & 1u) << n1;
  return g;
}
template <int R1, int R2>
__host__ __device__ constexpr unsigned split_second_mask(unsigned zm) {
  unsigned g = 0;
  for (int n2 = 0; n2 < R2; ++n2) g |= (split_group_mask<R1, R2>(zm, n2) == (1u << R1) - 1u ? 1u : 0u) << n2;
  return g;
}
template <int R1, int R2, int DIR, unsigned ZM, int N2>
__device__ __forceinline__ void dftz_split_first(float2* a, float2* b) {
  if constexpr (N2 < R2) {
    constexpr int R = R1 * R2;
    constexpr unsigned g = split_group_mask<R1, R2>(ZM, N2);
    float2 t[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) t[n1] = a[R2 * n1 + N2];
    DFTZ<R1, DIR, g>::run(t);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      if constexpr (g == (1u << R1) - 1u) b[N2 * R1 + k1] = make_float2(0.f, 0.f);
      else b[N2 * R1 + k1] = mul_root48<DIR>(t[k1], ((N2 * k1) % R) * (48 / R));
    }
    dftz_split_first<R1, R2, DIR, ZM, N2 + 1>(a, b);
  }
}
template <int R1, int R2, int DIR, unsigned ZM>
__device__ __forceinline__ void dftz_split(float2* a) {
  constexpr unsigned m2 = split_second_mask<R1, R2>(ZM);
  float2 b[R1 * R2];
  dftz_split_first<R1, R2, DIR, ZM, 0>(a, b);
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    float2 t[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) t[n2] = b[n2 * R1 + k1];
    DFTZ<R2, DIR, m2>::run(t);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) a[k1 + R1 * k2] = t[k2];
  }
}
template <int DIR, unsigned ZM>
struct DFTZ<6, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) { dftz_split<2, 3, DIR, ZM>(a); }
};
template <int DIR, unsigned ZM>
struct DFTZ<8, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) { dftz_split<2, 4, DIR, ZM>(a); }
};
template <int DIR, unsigned ZM>
struct DFTZ<12, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) { dftz_split<4, 3, DIR, ZM>(a); }
};
template <int DIR, unsigned ZM>
struct DFTZ<16, DIR, ZM> {
  __device__ __forceinline__ static void run(float2* a) { dftz_split<4, 4, DIR, ZM>(a); }
};

// ------------------------------------------------------------------ per-length schedules
// R0 == R_last wherever possible so inverse->pointwise->forward stays in registers.
template <int L>
struct Cfg;
#define NLV_CFG(L_, E_, NP_, A_, B_, C_, D_)                    \
  template <>                                                   \
  struct Cfg<L_> {                                              \
    static constexpr int L = L_, E = E_, T = L_ / E_, NP = NP_; \
    static constexpr int R0 = A_, R1 = B_, R2 = C_, R3 = D_;    \
  };
NLV_CFG(16, 4, 2, 4, 4, 1, 1)
NLV_CFG(32, 8, 2, 8, 4, 1, 1)
NLV_CFG(48, 12, 2, 12, 4, 1, 1)
NLV_CFG(64, 8, 2, 8, 8, 1, 1)
NLV_CFG(96, 24, 2, 12, 8, 1, 1)
NLV_CFG(128, 16, 2, 16, 8, 1, 1)
NLV_CFG(192, 24, 3, 8, 3, 8, 1)
NLV_CFG(256, 16, 2, 16, 16, 1, 1)
NLV_CFG(384, 24, 3, 8, 6, 8, 1)
NLV_CFG(512, 16, 3, 8, 8, 8, 1)
NLV_CFG(768, 24, 3, 8, 12, 8, 1)
NLV_CFG(1024, 32, 3, 16, 4, 16, 1)
#undef NLV_CFG

template <int L>
struct Sched {
  using C = Cfg<L>;
  static constexpr int RL = (C::NP == 4) ? C::R3 : (C::NP == 3) ? C::R2 : C::R1;  // radix of the last pass
  static constexpr bool kSymmetric = (C::R0 == RL);
  // index of register e in the pass-0 input pattern
  __device__ __forceinline__ static int in_idx(int t, int e) {
    return t + C::T * (e / C::R0) + (e % C::R0) * (L / C::R0);
  }
  // index of register e in the last pass's output pattern
  __device__ __forceinline__ static int out_idx(int t, int e) {
    return t + C::T * (e / RL) + (e % RL) * (L / RL);
  }
  // compile-time part of in/out index (t excluded)
  static constexpr int in_off(int e) { return C::T * (e / C::R0) + (e % C::R0) * (L / C::R0); }
  static constexpr int out_off(int e) { return C::T * (e / RL) + (e % RL) * (L / RL); }
};

// Inter-pass twiddle table, one block per pass p >= 1 (NS = R0 ... R_{p-1} points already combined, radix
// R = R_p), laid out [r - 1][k]: entry tw_base(NS) + (r - 1) NS + k = e^{-2 pi i k r / (NS R)}, k < NS,
// 1 <= r < R. Threads of a row transform hold consecutive k, so a warp's twiddle loads hit consecutive
// words (conflict-free) instead of the stride k r L / (NS R) of a plain e^{-2 pi i m / L} table (up to
// 16-way bank conflicts). At most L entries for every schedule here; built on the host (nlinv_plan_create).
template <int L>
__host__ __device__ constexpr int tw_base(int NS) {
  using C = Cfg<L>;
  const int Rs[4] = {C::R0, C::R1, C::R2, C::R3};
  int base = 0, ns = C::R0;
  for (int p = 1; p < C::NP; ++p) {
    if (ns == NS) return base;
    base += ns * (Rs[p] - 1);
    ns *= Rs[p];
  }
  return base;
}

// Twiddle from the shared table (entry m); DIR = +1 conjugates.
template <int DIR>
__device__ __forceinline__ float2 twid(const float2* tw, int m) {
  float2 w = tw[m];
  return DIR < 0 ? w : make_float2(w.x, -w.y);
}

// One Stockham pass on registers that hold this pass's input pattern.
template <int L, int R, int NS, int DIR>
__device__ __forceinline__ void pass_compute(float2* v, int t, const float2* tw) {
  using C = Cfg<L>;
  constexpr int E = C::E, T = C::T;
#pragma unroll
  for (int m = 0; m < E / R; ++m) {
    if (NS > 1) {
      const int j = t + T * m;
      const int k = j % NS;
#pragma unroll
      for (int r = 1; r < R; ++r) v[m * R + r] = cmul(v[m * R + r], twid<DIR>(tw, tw_base<L>(NS) + (r - 1) * NS + k));
    }
    DFT<R, DIR>::run(&v[m * R]);
  }
}

// Store the output of pass (R, NS) to the exchange buffer, then load the input pattern of
// the next pass (radix RN). BUF provides operator()(int index) -> float2&. SYNC is a barrier
// covering every thread of the transform.
template <int L, int R, int NS, int RN, class BUF, class SYNC>
__device__ __forceinline__ void pass_exchange(float2* v, int t, BUF& buf, SYNC sync) {
  using C = Cfg<L>;
  constexpr int E = C::E, T = C::T;
  // the first exchange (NS == 1) may use a bank-conflict swizzle of the buffer (buf.first)
#pragma unroll
  for (int m = 0; m < E / R; ++m) {
    const int j = t + T * m;
    const int base = (j / NS) * NS * R + (j % NS);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (NS == 1) buf.template first_st<L>(base + r * NS, r & 1) = v[m * R + r];
      else if constexpr (NS == C::R0) buf.template mid<L>(base + r * NS) = v[m * R + r];
      else buf(base + r * NS) = v[m * R + r];
    }
  }
  sync();
#pragma unroll
  for (int m = 0; m < E / RN; ++m) {
#pragma unroll
    for (int r = 0; r < RN; ++r) {
      if constexpr (NS == 1) v[m * RN + r] = buf.template first_ld<L>(t + T * m + r * (L / RN));
      else if constexpr (NS == C::R0) v[m * RN + r] = buf.template mid<L>(t + T * m + r * (L / RN));
      else v[m * RN + r] = buf(t + T * m + r * (L / RN));
    }
  }
  sync();
}

// Full length-L transform: registers in pass-0 input pattern -> registers in last-pass
// output pattern. Unnormalised, X_k = sum_n x_n e^{DIR 2 pi i n k / L}.
// ZM0: bit r set if every register slot m*R0 + r of the pass-0 input is structurally zero
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// hook() runs once every thread is past the last shared-memory exchange (the buffer is free again,
// e.g. for an asynchronous bulk copy into it) while the last pass computes in registers
template <int L, int DIR, unsigned ZM0 = 0, class BUF, class SYNC, class HOOK = NoHook>
__device__ __forceinline__ void fft(float2* v, int t, const float2* tw, BUF& buf, SYNC sync, HOOK hook = HOOK{}) {
  using C = Cfg<L>;
  if constexpr (ZM0 == 0) {
    pass_compute<L, C::R0, 1, DIR>(v, t, tw);
  } else {
#pragma unroll
    for (int m = 0; m < C::E / C::R0; ++m) DFTZ<C::R0, DIR, ZM0>::run(&v[m * C::R0]);
  }
  pass_exchange<L, C::R0, 1, C::R1>(v, t, buf, sync);
  if constexpr (C::NP == 2) hook();
  pass_compute<L, C::R1, C::R0, DIR>(v, t, tw);
  if constexpr (C::NP >= 3) {
    pass_exchange<L, C::R1, C::R0, C::R2>(v, t, buf, sync);
    if constexpr (C::NP == 3) hook();
    pass_compute<L, C::R2, C::R0 * C::R1, DIR>(v, t, tw);
  }
  if constexpr (C::NP >= 4) {
    pass_exchange<L, C::R2, C::R0 * C::R1, C::R3>(v, t, buf, sync);
    hook();
    pass_compute<L, C::R3, C::R0 * C::R1 * C::R2, DIR>(v, t, tw);
  }
}

// Registers in output pattern -> registers in input pattern (no-op for symmetric schedules).
template <int L, class BUF, class SYNC>
__device__ __forceinline__ void out_to_in(float2* v, int t, BUF& buf, SYNC sync) {
  using S = Sched<L>;
  using C = Cfg<L>;
  if constexpr (!S::kSymmetric) {
#pragma unroll
    for (int e = 0; e < C::E; ++e) buf(S::out_idx(t, e)) = v[e];
    sync();
#pragma unroll
    for (int e = 0; e < C::E; ++e) v[e] = buf(S::in_idx(t, e));
    sync();
  }
}

}  // namespace nlv
