// csph_staged.cu -- the paper's kernel split K1..K8, one CUDA
// kernel per stage with every intermediate in HBM.  This is the straightforward
// GPU transcription of R used as the correctness baseline next to the fused
// y-marching kernel (csph_fused.cu).
#include "csph_internal.cuh"
#include "csph_launch.h"

namespace ck {

namespace {

struct Range {
  int i0, i1, j0, j1;
};

__device__ __forceinline__ bool in_range(const Range& r, int& i, int& j) {
  i = r.i0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  j = r.j0 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  return i < r.i1 && j < r.j1;
}

// K1: wet mask, eta, r, u, v on every padded cell
__global__ void k1_level0(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R, Phys P) {
  if (C->status) return;
  int i, j;
  if (!in_range(R, i, j)) return;
  const int p = C->parity;
  size_t c = off(S.pitch, i, j);
  double H = S.H[p][c];
  bool w = H > P.eps;
  T.eta[c] = H + S.b[p][c];
  T.w[c] = w ? 1 : 0;
  if (w) {
    double r = 1.0 / H;
    T.r[c] = r;
    T.u[c] = S.Qx[p][c] * r;
    T.v[c] = S.Qy[p][c] * r;
  } else {
    T.r[c] = 0.0; T.u[c] = 0.0; T.v[c] = 0.0;
  }
}

// K2: forces at t_n and Manning gamma
__global__ void k2_forces(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R, Phys P) {
  if (C->status) return;
  int i, j;
  if (!in_range(R, i, j)) return;
  const int p = C->parity;
  size_t c = off(S.pitch, i, j);
  if (!T.w[c]) { T.phix[c] = 0.0; T.phiy[c] = 0.0; T.gam[c] = 0.0; return; }
  const double* b = S.b[p];
  size_t e = c + 1, wv = c - 1, n = c + S.pitch, s = c - S.pitch;
  double PE = face_force(P.cPh, T.eta[c], b[c], T.eta[e], b[e]);
  double PW = face_force(P.cPh, T.eta[wv], b[wv], T.eta[c], b[c]);
  double PN = face_force(P.cPh, T.eta[c], b[c], T.eta[n], b[n]);
  double PS = face_force(P.cPh, T.eta[s], b[s], T.eta[c], b[c]);
  T.phix[c] = -(PE + PW);
  T.phiy[c] = -(PN + PS);
  if (S.cg) {  // NEXT-3 Manning field
    double u = T.u[c], v = T.v[c];
    double sp = sqrt0(u * u + v * v);
    T.gam[c] = (S.cg[c] * sp) * (T.r[c] * icbrt(S.H[p][c]));
  } else if (P.fric) {
    double u = T.u[c], v = T.v[c];
    double sp = sqrt0(u * u + v * v);
    T.gam[c] = (P.cgam * sp) * (T.r[c] * icbrt(S.H[p][c]));
  } else {
    T.gam[c] = 0.0;
  }
}

// K4: predictor to t_{n+1/2}
__global__ void k4_predictor(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R,
                             Phys P) {
  if (C->status) return;
  int i, j;
  if (!in_range(R, i, j)) return;
  const int p = C->parity;
  size_t c = off(S.pitch, i, j);
  double H = S.H[p][c];
  if (!T.w[c]) { T.Hh[c] = H; T.ut[c] = 0.0; T.vt[c] = 0.0; return; }
  const double theta = 0.5 * C->tau;
  double div = ((T.u[c + 1] - T.u[c - 1]) + (T.v[c + S.pitch] - T.v[c - S.pitch])) * P.inv_2h;
  T.Hh[c] = H * fma(-theta, div, 1.0);
  double f = 1.0 / fma(theta, T.gam[c], 1.0);
  T.ut[c] = (fma(theta, T.phix[c], S.Qx[p][c]) * f) * T.r[c];
  T.vt[c] = (fma(theta, T.phiy[c], S.Qy[p][c]) * f) * T.r[c];
}

// K5: forces at t_{n+1/2}
__global__ void k5_forces_half(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R,
                               Phys P) {
  if (C->status) return;
  int i, j;
  if (!in_range(R, i, j)) return;
  const int p = C->parity;
  size_t c = off(S.pitch, i, j);
  if (!T.w[c]) { T.phix2[c] = 0.0; T.phiy2[c] = 0.0; return; }
  const double* b = S.b[p];
  const double* Hh = T.Hh;
  size_t e = c + 1, wv = c - 1, n = c + S.pitch, s = c - S.pitch;
  double ec = Hh[c] + b[c];
  double PE = face_force(P.cPh, ec, b[c], Hh[e] + b[e], b[e]);
  double PW = face_force(P.cPh, Hh[wv] + b[wv], b[wv], ec, b[c]);
  double PN = face_force(P.cPh, ec, b[c], Hh[n] + b[n], b[n]);
  double PS = face_force(P.cPh, Hh[s] + b[s], b[s], ec, b[c]);
  T.phix2[c] = -(PE + PW);
  T.phiy2[c] = -(PN + PS);
}

// K6: corrector momenta Q^L; per-cell Grass flux J0 for K7
__global__ void k6_corrector(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R,
                             Range RJ, Phys P) {
  if (C->status) return;
  int i, j;
  const int p = C->parity;
  // J0 on the wider range RJ (the grid is sized for RJ)
  if (in_range(RJ, i, j)) {
    size_t c = off(S.pitch, i, j);
    double jx, jy, ja;
    const double Hc = S.H[p][c];
    grass_gated(P, T.ut[c], T.vt[c], Hc, cell_aj(P, S, c, Hc), jx, jy, ja);
    T.J0x[c] = jx; T.J0y[c] = jy; T.J0a[c] = ja;
  }
  if (i < R.i0 || i >= R.i1 || j < R.j0 || j >= R.j1) return;
  size_t c = off(S.pitch, i, j);
  if (!T.w[c]) { T.QLx[c] = 0.0; T.QLy[c] = 0.0; return; }
  const double tau = C->tau;
  double f = 1.0 / fma(tau, T.gam[c], 1.0);
  T.QLx[c] = fma(tau, T.phix2[c], S.Qx[p][c]) * f;
  T.QLy[c] = fma(tau, T.phiy2[c], S.Qy[p][c]) * f;
}

// K7: one face per thread. axis 0: face between (i-1,j),(i,j).
template <int AXIS>
__global__ void k7_fluxes(StripView S, const Ctrl* __restrict__ C, Scratch T, Range R, Phys P) {
  if (C->status) return;
  int i, j;
  if (!in_range(R, i, j)) return;
  const int p = C->parity;
  const size_t st = AXIS == 0 ? 1 : (size_t)S.pitch;
  size_t Rc = off(S.pitch, i, j), Lc = Rc - st;
  double* FH = AXIS == 0 ? T.FH : T.GH;
  double* FQn = AXIS == 0 ? T.FQx : T.GQy;
  double* FQt = AXIS == 0 ? T.FQy : T.GQx;
  double* FJ = AXIS == 0 ? T.FJ : T.GJ;
  if (!T.w[Lc] && !T.w[Rc]) {
    FH[Rc] = 0.0; FQn[Rc] = 0.0; FQt[Rc] = 0.0; FJ[Rc] = 0.0;
    return;
  }
  const double* H = S.H[p];
  const double* un = AXIS == 0 ? T.ut : T.vt;
  const double* ut = AXIS == 0 ? T.vt : T.ut;
  size_t LL = Lc - st, RR = Rc + st;
  const double* q[4] = {T.eta, H, un, ut};
  double qm[4], qp[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double sL = minmod(q[k][Lc] - q[k][LL], q[k][Rc] - q[k][Lc]);
    double sR = minmod(q[k][Rc] - q[k][Lc], q[k][RR] - q[k][Rc]);
    qm[k] = fma(0.5, sL, q[k][Lc]);   // face states with one rounding
    qp[k] = fma(-0.5, sR, q[k][Rc]);
  }
  double F0, F1, F2;
  hll_face(P.g, qm[0], qm[1], qm[2], qm[3], qp[0], qp[1], qp[2], qp[3], F0, F1, F2);
  FH[Rc] = F0; FQn[Rc] = F1; FQt[Rc] = F2;
  const double* Jn = AXIS == 0 ? T.J0x : T.J0y;
  const double* b = S.b[p];
  FJ[Rc] = sed_face(P, un[Lc], un[Rc], Jn[Lc], Jn[Rc], T.J0a[Lc], T.J0a[Rc], b[Lc], b[Rc]);
}

// K8: conservative update, dry-momentum zeroing, negative-depth flag,
// next-step Eq.7 maxima.
__global__ void k8_update(StripView S, Ctrl* C, Scratch T, Range R, Phys P,
                          unsigned long long* gM) {
  if (C->status) return;
  int i, j;
  bool ok = in_range(R, i, j);
  const int p = C->parity, q = p ^ 1;
  unsigned long long m0 = 0, m1 = 0, m2 = 0;
  if (ok) {
    const double tau = C->tau;
    const double lam = tau / P.h;
    size_t c = off(S.pitch, i, j), e = c + 1, n = c + S.pitch;
    double W = S.W ? S.W[c] : S.Wc;
    double dH = (T.FH[e] - T.FH[c]) + (T.GH[n] - T.GH[c]);
    double dQx = (T.FQx[e] - T.FQx[c]) + (T.GQx[n] - T.GQx[c]);
    double dQy = (T.FQy[e] - T.FQy[c]) + (T.GQy[n] - T.GQy[c]);
    double dJ = (T.FJ[e] - T.FJ[c]) + (T.GJ[n] - T.GJ[c]);
    double Hn = fma(-lam, dH, S.H[p][c]);
    double Qxn = fma(-lam, dQx, T.QLx[c]);
    double Qyn = fma(-lam, dQy, T.QLy[c]);
    double bn = fma(-(lam * W), dJ, S.b[p][c]) + (tau * W) * P.src;
    apply_sources(S, tau, c, Hn, Qxn, Qyn);
    bool wet = Hn > P.eps;
    if (!wet) { Qxn = 0.0; Qyn = 0.0; }
    if (Hn < -P.neg_tol) atomicMax(&gM[3], 1ull);  // combined like the maxima
    S.H[q][c] = Hn; S.Qx[q][c] = Qxn; S.Qy[q][c] = Qyn; S.b[q][c] = bn;
    if (wet) {
      double t1, t2, t3;
      dt_terms(P, Hn, Qxn, Qyn, W, cell_aj(P, S, c, Hn), t1, t2, t3);
      m0 = dbits(t1); m1 = dbits(t2); m2 = dbits(t3);
    }
  }
  block_max3_atomic<8>(m0, m1, m2, gM);
}

}  // namespace

void launch_staged_step(const StripView& S, Ctrl* C, const Scratch& T, const Phys& P,
                        unsigned long long* gM, cudaStream_t st, long long* nlaunch) {
  const int nx = S.nx, ny = S.ny;
  dim3 blk(32, 8);
  auto grid_for = [&](const Range& r) {
    return dim3((unsigned)((r.i1 - r.i0 + 31) / 32), (unsigned)((r.j1 - r.j0 + 7) / 8));
  };
  Range r3{-3, nx + 3, -3, ny + 3}, r2{-2, nx + 2, -2, ny + 2}, r1{-1, nx + 1, -1, ny + 1},
      r0{0, nx, 0, ny};
  k1_level0<<<grid_for(r3), blk, 0, st>>>(S, C, T, r3, P);
  k2_forces<<<grid_for(r2), blk, 0, st>>>(S, C, T, r2, P);
  k4_predictor<<<grid_for(r2), blk, 0, st>>>(S, C, T, r2, P);
  k5_forces_half<<<grid_for(r1), blk, 0, st>>>(S, C, T, r1, P);
  // K6 grid covers the J0 range r2 (Q^L on r0 inside it)
  {
    Range rj = r2;
    k6_corrector<<<grid_for(rj), blk, 0, st>>>(S, C, T, r0, rj, P);
  }
  Range fx{0, nx + 1, 0, ny}, fy{0, nx, 0, ny + 1};
  k7_fluxes<0><<<grid_for(fx), blk, 0, st>>>(S, C, T, fx, P);
  k7_fluxes<1><<<grid_for(fy), blk, 0, st>>>(S, C, T, fy, P);
  k8_update<<<grid_for(r0), blk, 0, st>>>(S, C, T, r0, P, gM);
  *nlaunch += 8;
}

}  // namespace ck
