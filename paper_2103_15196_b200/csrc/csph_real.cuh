// csph_real.cuh -- the fused kernel's arithmetic helpers, generic in the real type T.
// T = double: the same operations, in the same order, as csph_internal.cuh (reading R,
// bitwise parity with the oracle).  T = float: the NEXT-2 fp32 mode,
// which uses the hardware's correctly rounded fp32 reciprocal and square root.
#pragma once

#include "csph_internal.cuh"

namespace ck {

// Scalar constants of R converted once to T at kernel start.
template <typename T>
struct PT {
  T g, eps, neg_tol, A_J, C_J, C_Sh, kappa, cPh, cgam, inv_h, inv_2h, src, d50, hbm;
  int m_grass, fric, transport;
  double m_real;
};

template <typename T>
__device__ __forceinline__ PT<T> make_pt(const Phys& P) {
  PT<T> q;
  q.g = T(P.g); q.eps = T(P.eps); q.neg_tol = T(P.neg_tol); q.A_J = T(P.A_J);
  q.C_J = T(P.C_J); q.C_Sh = T(P.C_Sh); q.kappa = T(P.kappa); q.cPh = T(P.cPh);
  q.cgam = T(P.cgam); q.inv_h = T(P.inv_h); q.inv_2h = T(P.inv_2h); q.src = T(P.src);
  q.d50 = T(P.d50);
  q.hbm = T(P.hbm);
  q.m_grass = P.m_grass; q.fric = P.fric; q.transport = P.transport;
  q.m_real = P.m_real;
  return q;
}

// Opaque copy of a 0/1 flag: stops the compiler from folding "x > c || y > c" into
// "fmax(x, y) > c", which sm_100 has no fp64 instruction for (an 8-instruction emulation
// instead of two compares).
__device__ __forceinline__ unsigned opq(unsigned x) {
  unsigned y;
  asm("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
template <typename T> __device__ __forceinline__ unsigned gt_u(T x, T c) { return opq(x > c ? 1u : 0u); }

template <typename T> __device__ __forceinline__ T smin_t(T a, T b) { return (a < b) ? a : b; }
template <typename T> __device__ __forceinline__ T smax_t(T a, T b) { return (a > b) ? a : b; }

// minmod of R without branches: for a, b both > 0 R's min(a, b) = (a < b ? a : b) and for
// both < 0 R's max(a, b) = (a > b ? a : b) are the same selection (|a| < |b| ? a : b); all
// other cases (opposite signs, a zero, a NaN) give +0.  Bitwise identical to R.
template <typename T>
__device__ __forceinline__ T minmod_t(T a, T b) {
  const bool same = ((a > T(0)) & (b > T(0))) | ((a < T(0)) & (b < T(0)));
  const T pick = (fabs(a) < fabs(b)) ? a : b;
  return same ? pick : T(0);
}
// fp64: the same value with two fp64 compares instead of five.  pick is the operand of
// smaller magnitude, so pick != 0 <=> both are nonzero; equal sign bits (integer test on
// the high words) then means both > 0 or both < 0.  Identical to R for every non-NaN a, b
// (a NaN slope only arises from a non-finite state, which Eq.7 reports as ENONFINITE).
template <>
__device__ __forceinline__ double minmod_t<double>(double a, double b) {
  const double pick = (fabs(a) < fabs(b)) ? a : b;
  const bool same = ((__double2hiint(a) ^ __double2hiint(b)) >= 0) & (pick != 0.0);
  return same ? pick : 0.0;
}

__device__ __forceinline__ double rcp_t(double x) { return rcp_nb(x); }
__device__ __forceinline__ float rcp_t(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double sqrt0_t(double x) { return sqrt0nb(x); }
__device__ __forceinline__ float sqrt0_t(float x) { return x > 0.0f ? __fsqrt_rn(x) : x; }
// sqrt of g*H for a wet depth: in the hot specialisation g*eps_dry >= 2^-890 (launch_v),
// so the argument is a normal number >= 2^-890 and the plain fast path is exact
template <bool GEN> __device__ __forceinline__ double sqrt_gh_t(double x) {
  return GEN ? sqrt0nb(x) : sqrt_nb(x);
}
template <bool GEN> __device__ __forceinline__ float sqrt_gh_t(float x) { return sqrt0_t(x); }
__device__ __forceinline__ double icbrt_t(double x) { return icbrt(x); }
// fp32 x^(-1/3): bit-trick seed and 3 Newton steps (fp32 mode only)
__device__ __forceinline__ float icbrt_t(float x) {
  float y = __int_as_float(0x54A2FA8C - __float_as_int(x) / 3);
  const float third = 1.0f / 3.0f;
#pragma unroll
  for (int k = 0; k < 3; ++k) y = fmaf(y, fmaf(-x, (y * y) * y, 1.0f) * third, y);
  return y;
}
__device__ __forceinline__ unsigned long long dbits_t(double x) { return dbits(x); }
__device__ __forceinline__ unsigned long long dbits_t(float x) { return dbits((double)x); }

// K2/K5 face force (hydrostatic form): (c_P/2 (H*_L + H*_R)) (H*_R - H*_L)
template <typename T>
__device__ __forceinline__ T face_force_t(T cPh, T etaL, T bL, T etaR, T bR) {
  T bs = smax_t(bL, bR);
  T hL = smax_t(T(0), etaL - bs);
  T hR = smax_t(T(0), etaR - bs);
  return (cPh * (hL + hR)) * (hR - hL);
}

template <bool GEN, typename T>
__device__ __forceinline__ T pow_m_t(int m, double mr, T s2, T a) {
  if (!GEN) return s2;
  if constexpr (sizeof(T) == 8) {
    if (mr >= 0.0) return pow_pinned(s2, 0.5 * mr);  // NEXT-4 real exponent (fp64 only)
  }
  if (m == 2) return s2;
  T pw = T(1);
  for (int k = 0; k < m / 2; ++k) pw = pw * s2;
  if (m & 1) pw = pw * a;
  return pw;
}

template <bool GEN, typename T>
__device__ __forceinline__ void grass_t(const PT<T>& P, T ut, T vt, T H, T A, T& jx, T& jy,
                                        T& ja) {
  T s2 = ut * ut + vt * vt;
  T sa = sqrt0_t(s2);
  T a = A * pow_m_t<GEN>(P.m_grass, P.m_real, s2, sa);
  // Eq.5 gate and reading #31: no bedload through a film (H <= h_bed_min, default d50)
  const bool gate = ((P.C_Sh == T(0)) | ((s2 * s2) * s2 > P.kappa * H)) & (H > P.hbm);
  jx = gate ? a * ut : T(0); jy = gate ? a * vt : T(0); ja = gate ? a * sa : T(0);
}

template <typename T>
__device__ __forceinline__ T sed_face_t(const PT<T>& P, T unL, T unR, T JnL, T JnR, T JaL, T JaR,
                                        T bL, T bR) {
  const T us = unL + unR;
  const bool up = us > T(0), dn = us < T(0);
  const T Jn = up ? JnL : (dn ? JnR : T(0.5) * (JnL + JnR));
  const T Ja = up ? JaL : (dn ? JaR : T(0.5) * (JaL + JaR));
  return fma(-(P.C_J * Ja), (bR - bL) * P.inv_h, Jn);
}

template <bool GEN, typename T>
__device__ __forceinline__ void dt_terms_t(const PT<T>& P, T H, T Qx, T Qy, T W, T A, T& t1,
                                           T& t2, T& t3) {
  T r = rcp_t(H);
  T u = Qx * r, v = Qy * r;
  T s2 = u * u + v * v;
  T a = sqrt0_t(s2);
  t1 = s2;
  t2 = a + sqrt_gh_t<GEN>(P.g * H);
  bool gate = ((P.C_Sh == T(0)) || ((s2 * s2) * s2 > P.kappa * H)) && (H > P.hbm);
  t3 = gate ? ((A * pow_m_t<GEN>(P.m_grass, P.m_real, s2, a)) * a) * W : T(0);
}

// Wall-only ghost writer (the hot-path specialisation), generic in T.
template <typename T>
__device__ __forceinline__ void write_wall_ghosts_t(const StripView& S, T* oH, T* oQx, T* oQy,
                                                    T* ob, int col, int j, T Hn, T Qxn, T Qyn,
                                                    T bn, bool gx) {
  const size_t o = off(S.pitch, col, j);
  oH[o] = Hn; oQx[o] = Qxn; oQy[o] = Qyn; ob[o] = bn;
  const bool gyl = S.wall_lo && j < 3, gyh = S.wall_hi && j >= S.ny - 3;
  if (!(gx || gyl || gyh)) return;
  const int gcs[2] = {col < 3 ? -1 - col : INT_MIN, col >= S.nx - 3 ? 2 * S.nx - 1 - col : INT_MIN};
  const int grs[2] = {gyl ? -1 - j : INT_MIN, gyh ? 2 * S.ny - 1 - j : INT_MIN};
  for (int a = 0; a < 2; ++a) {
    if (gcs[a] == INT_MIN) continue;
    const size_t g = off(S.pitch, gcs[a], j);
    oH[g] = Hn; oQx[g] = -Qxn; oQy[g] = Qyn; ob[g] = bn;
  }
  for (int c = 0; c < 2; ++c) {
    if (grs[c] == INT_MIN) continue;
    size_t g = off(S.pitch, col, grs[c]);
    oH[g] = Hn; oQx[g] = Qxn; oQy[g] = -Qyn; ob[g] = bn;
    for (int a = 0; a < 2; ++a) {
      if (gcs[a] == INT_MIN) continue;
      g = off(S.pitch, gcs[a], grs[c]);
      oH[g] = Hn; oQx[g] = -Qxn; oQy[g] = -Qyn; ob[g] = bn;
    }
  }
}

}  // namespace ck
