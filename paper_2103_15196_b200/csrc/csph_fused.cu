// csph_fused.cu -- one CUDA kernel per CSPH-TVD step (K1..K8 of PAPER.md:224-238 fused).
//
// Design:
//  * A CTA owns a column tile of TX = NT - 8 output cells and marches down a chunk of
//    TY rows ("2.5D" y-march).  Thread t owns padded column x0 - 4 + t for the whole march.
//  * Input rows (H, Qx, Qy, b [, W]) are staged into a D-slot shared-memory ring by 1D TMA
//    bulk copies (cp.async.bulk ... mbarrier::complete_tx), PF rows ahead of use.
//  * Every stage of R is computed once per cell: x-neighbour values are exchanged through
//    shared memory (two barriers per row), y-neighbour values are carried in registers.
//    The update of row L-3 is produced when row L is loaded (stencil radius 3).
//  * Epilogue: stores of (H, Qx, Qy, b) for row L-3, wall-mirror ghosts, the next step's
//    Eq.7 maxima (warp shuffle + block max + one atomicMax per CTA) and the negative-depth flag.
// The arithmetic per cell is the same sequence of IEEE operations as the oracle (-fmad=false).
#include <climits>
#include <cstdlib>

#include "csph_launch.h"
#include "csph_real.cuh"

#ifndef CSPH_UNROLL
#define CSPH_UNROLL 2
#endif

namespace ck {

namespace {

constexpr int kUnroll = CSPH_UNROLL;  // y-march unroll of the fp64 hot specialisation (register
                                      // renaming of the carried window: fewer moves, +1.6 %)
#ifndef CSPH_MINB32
#define CSPH_MINB32 5
#endif
constexpr int kMinB32 = CSPH_MINB32;  // resident CTAs per SM of the fp32 instance

#ifndef CSPH_PUSH
#define CSPH_PUSH 1  // development knob: halo push code compiled out (A/B)
#endif
#ifndef CSPH_GUARD
#define CSPH_GUARD 0
#endif
// warp-uniform guard: skip a stage when no lane of the warp needs it
#define ANYW(x) (CSPH_GUARD ? __any_sync(0xffffffffu, (x)) : true)
// friction / transport switches: runtime in the general (and fp32) instances, compile-time
// on in the fp64 hot-path specialisation (launch_v sends other cases to the general one)
#define FRIC (RTF ? P.fric != 0 : true)
#define TRANSP (RTF ? P.transport != 0 : true)

// Ring of D slots with rows prefetched PF ahead; rows L-4..L are live, so D >= PF + 5.

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_row(void* dst, const void* src, unsigned bytes,
                                        unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename T, int NT, bool HASW, int D>
struct Smem {
  static constexpr int NF = HASW ? 5 : 4;
  static constexpr int OFR = 16 / (int)sizeof(T);  // ring data offset: 16 B aligned
  static constexpr int RW = NT + 2 * OFR;          // ring row: data at [OFR, OFR+NT)
  static constexpr int XW = NT + 2;                // exchange row: element t at [t+1]
  alignas(128) T ring[D][NF][RW];
  T U[2][XW];      // u of the last two rows (div)
  T PE[XW];        // K2 x-face force (t|t+1), row L
  T X2[2][5][XW];  // K4 outputs by row parity: H_half, u~, v~, J0x, |J0|
  T X3[5][XW];     // row L-1: K5 x-face force, sigma_x (eta, H, u~, v~)
  T X4[4][XW];     // row L-1: x-face fluxes (t|t+1): F^H, F^Qx, F^Qy, F^J
  alignas(8) unsigned long long bar[D];
  unsigned long long red[3][NT / 32];
  unsigned wm[NT / 32];
#ifdef CSPH_SMEM_EXTRA
  char pad_[CSPH_SMEM_EXTRA];  // development knob: occupancy experiments
#endif
};

enum { F_H = 0, F_QX = 1, F_QY = 2, F_B = 3, F_W = 4 };

// K7 hydrostatic step + HLL without branches: every case of
// hll_face() is evaluated with the same operations and the result selected, so
// the value is bitwise identical.  Callers have already excluded both-dry cells.
#ifndef CSPH_HLL_FAST
#define CSPH_HLL_FAST 1
#endif
template <typename T>
__device__ __forceinline__ void hll_bf(T g, T eta_m, T H_m, T un_m, T ut_m, T eta_p, T H_p,
                                       T un_p, T ut_p, bool off, T& F0, T& F1, T& F2) {
  const T bs = smax_t(eta_m - H_m, eta_p - H_p);
  const T Hm = smax_t(T(0), eta_m - bs);
  const T Hp = smax_t(T(0), eta_p - bs);
  // wet flags of the two reconstructed sides (opaque: "both dry" stays two compares)
  const unsigned wm = gt_u(Hm, T(0)), wp = gt_u(Hp, T(0));
  const bool dp = wp == 0u;
  const T mm = Hm * un_m, mp = Hp * un_p;
  const T cm = sqrt0_t(g * Hm), cp = sqrt0_t(g * Hp);
  // the three wave-speed cases of R, all evaluated, then selected
  const T aL = un_m - cm, aR = un_p - cp, bL2 = un_m + cm, bR2 = un_p + cp;
  const bool both = (wm & wp) != 0u;
  const T fl1 = mm * un_m, fl2 = mm * ut_m, fr1 = mp * un_p, fr2 = mp * ut_p;
  const T d0 = Hp - Hm, d1 = mp - mm, d2 = Hp * ut_p - Hm * ut_m;
  if (CSPH_HLL_FAST && __all_sync(0xffffffffu, both & !off)) {
    // warp-uniform common case (both reconstructed sides wet, a face of a wet cell): R's
    // both-wet speeds without the dry-side selects; then, unless some lane is supercritical,
    // the HLL average without the upwind selects.  Same operations, same values.
    const T SL = smin_t(aL, aR), SR = smax_t(bL2, bR2);
    const T inv = rcp_t(SR - SL);
    const T SLSR = SL * SR;
    const T h0 = ((SR * mm - SL * mp) + SLSR * d0) * inv;
    const T h1 = ((SR * fl1 - SL * fr1) + SLSR * d1) * inv;
    const T h2 = ((SR * fl2 - SL * fr2) + SLSR * d2) * inv;
    const bool up = SL >= T(0), dn = SR <= T(0);
    if (__any_sync(0xffffffffu, up | dn)) {
      F0 = up ? mm : (dn ? mp : h0);
      F1 = up ? fl1 : (dn ? fr1 : h1);
      F2 = up ? fl2 : (dn ? fr2 : h2);
    } else {
      F0 = h0; F1 = h1; F2 = h2;
    }
    return;
  }
  const T SL = both ? smin_t(aL, aR) : (dp ? aL : fma(T(-2), cp, un_p));
  const T SR = both ? smax_t(bL2, bR2) : (dp ? fma(T(2), cm, un_m) : bR2);
  // both reconstructed sides dry, or a both-dry face of cells (off): the face carries 0
  const bool none = ((wm | wp) == 0u) | off;
  const T den = none ? T(1) : (SR - SL);
  const T inv = rcp_t(den);
  const T SLSR = SL * SR;
  const T h0 = ((SR * mm - SL * mp) + SLSR * d0) * inv;
  const T h1 = ((SR * fl1 - SL * fr1) + SLSR * d1) * inv;
  const T h2 = ((SR * fl2 - SL * fr2) + SLSR * d2) * inv;
  const bool up = SL >= T(0), dn = SR <= T(0);
  F0 = none ? T(0) : (up ? mm : (dn ? mp : h0));
  F1 = none ? T(0) : (up ? fl1 : (dn ? fr1 : h1));
  F2 = none ? T(0) : (up ? fl2 : (dn ? fr2 : h2));
}

template <typename T, int NT, bool HASW, int D, int PF, int MINB, bool GEN>
__global__ void __launch_bounds__(NT, MINB)
    fused_step_kernel(StripView S, Ctrl* __restrict__ C, Phys P,
                      unsigned long long* __restrict__ gM, int row0, int row1, int TY, Hgs hg) {
  static_assert(D >= PF + 5, "ring too shallow");
  constexpr int TX = NT - 8;
  using SM = Smem<T, NT, HASW, D>;
  static_assert(!GEN || sizeof(T) == 8, "NEXT-3/4 features are fp64 only");
  constexpr bool RTF = GEN || sizeof(T) == 4;
  extern __shared__ __align__(128) unsigned char smraw[];
  SM& sm = *reinterpret_cast<SM*>(smraw);

  const int status = C->status;
  if (status) return;
  const int par = C->parity;
  const PT<T> Q = make_pt<T>(P);
  const double taud = C->tau;
  const T tau = T(taud);
  const T theta = T(0.5) * tau;
  const T lam = T(taud / P.h);  // lambda in fp64 (identical for T = double)
  // state buffers hold T values (fp32 mode reuses the fp64 allocations)
  auto tp = [](double* x) { return reinterpret_cast<T*>(x); };
  // A_J of a cell: constant, or Eq.4 per cell (NEXT-4, fp64 GEN instance only)
  auto aj_at = [&](size_t c, T Hc) -> T {
    if constexpr (GEN) return cell_aj(P, S, c, Hc);
    else return Q.A_J;
  };
  const T* __restrict__ gin[5] = {tp(par ? S.H[1] : S.H[0]), tp(par ? S.Qx[1] : S.Qx[0]),
                                       tp(par ? S.Qy[1] : S.Qy[0]), tp(par ? S.b[1] : S.b[0]),
                                  reinterpret_cast<const T*>(S.W)};
  T* __restrict__ oH = tp(par ? S.H[0] : S.H[1]);
  T* __restrict__ oQx = tp(par ? S.Qx[0] : S.Qx[1]);
  T* __restrict__ oQy = tp(par ? S.Qy[0] : S.Qy[1]);
  T* __restrict__ ob = tp(par ? S.b[0] : S.b[1]);

  const int t = threadIdx.x;
  const int nx = S.nx, pitch = S.pitch;
  // the tile of this CTA: the launch's order list (costliest first), else natural order
  const int gx = (S.nx + TX - 1) / TX;
  const int lin = hg.order ? hg.order[blockIdx.x] : (int)blockIdx.x;
  const int bx = lin % gx, by = lin / gx;
  const int x0 = bx * TX;
  const int col = x0 - 4 + t;
  const int y0 = row0 + by * TY;
  const int y1 = min(y0 + TY, row1);
  if (y0 >= y1) return;
  // ---- HGS.  Under R a dry cell whose 4
  // edge neighbours are dry updates to the identity: its 4 faces are both-dry (no flux, no
  // sediment flux), Q^L = 0, so H' = H - lam*0, Q' = +0, b' = b - (lam W)*0 + (tau W)*src.
  // A tile is therefore an identity when no cell of it and no cell of the facing 1-cell
  // bands of its 4 edge neighbours was wet after the previous step (band-mask flags). ----
  // index of a static per-cell field (NEXT-3/4, GEN instance) at column c, row r, for a
  // read whose result may feed nothing: threads past the last ghost column of the last tile
  // and the phase A run one row beyond the march are clamped into the allocation
  auto fidx = [&](int c, int r) -> size_t {
    return off(pitch, min(c, nx + GX - 1), min(r, S.ny + GY - 1));
  };
  const int tr = y0 / TY;
  const int ti = tr * hg.ntx + bx;
  // HGS flags of a tile row facing a neighbouring strip go into its ghost flag rows too
  // (halo push): my first tile row to the strip below, my last to the one above
  auto push_flags = [&](unsigned m) {
    const size_t g = 2 * (size_t)hg.ntx * (size_t)(par ^ 1) + (size_t)bx;
    if (tr == 0 && S.ngflag[0]) S.ngflag[0][g + hg.ntx] = (unsigned char)m;
    if (tr == hg.nty - 1 && S.ngflag[1]) S.ngflag[1][g] = (unsigned char)m;
  };
  // ... and its rows 0..2 / ny-3..ny-1 into the neighbour's ghost rows: once the tile is done
  // (callers sit behind a barrier), the tile copies them -- with the x-ghost columns the first
  // and last tile columns wrote -- from its output buffer, outside the march's hot loop
  auto push_rows = [&]() {
    if constexpr (CSPH_PUSH) {
      const int q = par ^ 1;
      const int c0 = bx == 0 ? -GX : bx * TX;
      const int c1 = bx * TX + TX >= S.nx ? S.nx + GY : bx * TX + TX;
      const T* src[4] = {tp(q ? S.H[1] : S.H[0]), tp(q ? S.Qx[1] : S.Qx[0]),
                         tp(q ? S.Qy[1] : S.Qy[0]), tp(q ? S.b[1] : S.b[0])};
      bool pushed = false;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (!S.nH[side][q]) continue;
        const int ja = side == 0 ? y0 : max(y0, S.ny - GY);
        const int jb = side == 0 ? min(y1, GY) : y1;
        if (ja >= jb) continue;
        T* dst[4] = {tp(S.nH[side][q]), tp(S.nQx[side][q]), tp(S.nQy[side][q]),
                     tp(S.nb[side][q])};
        for (int j = ja; j < jb; ++j)
          for (int c = c0 + (int)threadIdx.x; c < c1; c += NT) {
            const size_t o = off(S.pitch, c, j);
            const long long r = (long long)o + S.ndel[side];
#pragma unroll
            for (int f = 0; f < 4; ++f) dst[f][r] = src[f][o];
          }
        pushed = true;
      }
      if (pushed || ((tr == 0 || tr == hg.nty - 1) && (S.ngflag[0] || S.ngflag[1])))
        __threadfence_system();  // visible to the peer before this grid completes
    }
  };
  // across an interior strip edge the facing tile row is the neighbouring strip's, whose
  // flags arrive with the halo rows (hg.glo / hg.ghi); without them such a tile marches
  if (hg.enable && (S.wall_lo || y0 > 0 || hg.glo) && (S.wall_hi || y1 < S.ny || hg.ghi)) {
    auto fl = [&](int r, int q) -> unsigned {
      if (q < 0 || q >= hg.ntx) return 0u;
      if (r < 0) return hg.glo ? hg.glo[q] : 0u;          // a wall brings no water
      if (r >= hg.nty) return hg.ghi ? hg.ghi[q] : 0u;
      return hg.fprev[r * hg.ntx + q];
    };
    const int q0 = bx;
    const bool dry = !(fl(tr, q0) & HGS_ANY) && !(fl(tr - 1, q0) & HGS_BOT) &&
                     !(fl(tr + 1, q0) & HGS_TOP) && !(fl(tr, q0 - 1) & HGS_RIGHT) &&
                     !(fl(tr, q0 + 1) & HGS_LEFT);
    if (dry) {
      const unsigned char stt = hg.tstate[ti];
      if (stt < 2 || Q.src != T(0) || S.beta) {
        // identity update: H' = H, Q' = +0, b' with R's K8 formula at zero fluxes (with
        // NEXT-3 sources H' = (H + tau s)/(1 + tau beta): a dry cell may become wet)
        const bool outc = (t >= 4) && (t < 4 + TX) && (col < nx);
        bool cwet = false;
        if (outc) {
          for (int j = y0; j < y1; ++j) {
            const size_t o = off(pitch, col, j);
            const T H3 = gin[0][o], b3 = gin[3][o];
            const T W3 = HASW ? gin[4][o] : T(S.Wc);
            const T z = T(0) + (T(0) - T(0));
            T Hn = fma(-lam, z, H3);
            T Qn = fma(-lam, z, T(0)), Qm = Qn;
            const T bn = fma(-(lam * W3), z, b3) + (tau * W3) * Q.src;
            if constexpr (GEN) apply_sources(S, tau, o, Hn, Qn, Qm);
            if (Hn > Q.eps) cwet = true;  // momenta stay +0 (they were +0 * a)
            if constexpr (GEN)
              write_with_ghosts(S, oH, oQx, oQy, ob, col, j, Hn, Qn, Qn, bn, feeds_xghost(S, col));
            else
              write_wall_ghosts_t(S, oH, oQx, oQy, ob, col, j, Hn, Qn, Qn, bn, feeds_xghost(S, col));
          }
        }
        const bool any = __syncthreads_or(cwet);
        if (t == 0) {
          if (hg.cost) hg.cost[ti] = 0;
          hg.tstate[ti] = any ? 0 : (unsigned char)(stt + 1);
          hg.fnext[ti] = any ? HGS_ALL : 0;  // conservative: every band
          push_flags(any ? HGS_ALL : 0);
          atomicAdd(&hg.stats[1], 1ull);
        }
        push_rows();  // after __syncthreads_or: every thread's rows are written
        // a cell made wet by a source has Q' = +0: its Eq.7 terms are those of a
        // still wet cell
        if (cwet) {
          for (int j = y0; j < y1; ++j) {
            const size_t o = off(pitch, col, j);
            const T Hn = oH[o];
            if (Hn > Q.eps) {
              T t1, t2, t3;
              dt_terms_t<GEN>(Q, Hn, T(0), T(0), HASW ? gin[4][o] : T(S.Wc),
                            aj_at(o, Hn), t1, t2, t3);
              unsigned long long a2 = dbits_t(t1), b2 = dbits_t(t2), c2 = dbits_t(t3);
              atomicMax(&gM[0], a2); atomicMax(&gM[1], b2); atomicMax(&gM[2], c2);
            }
          }
        }
        return;
      }
      if (t == 0) {
        atomicAdd(&hg.stats[2], 1ull);
        hg.fnext[ti] = 0;
        push_flags(0);
        if (tr == 0 || tr == hg.nty - 1) __threadfence_system();
        if (hg.cost) hg.cost[ti] = 0;
      }
      return;  // both buffers already hold the identity (tstate >= 2, no source)
    }
  }
  const int rfirst = y0 - GY;       // first input row
  const int niter = (y1 + 2) - rfirst + 1;  // input rows y0-3 .. y1+2
  // columns copied per row: [x0-4, min(x0-4+NT, nx+4)), even count
  int ncopy = min(NT, nx + 8 - x0);
  ncopy = (ncopy + SM::OFR - 1) & ~(SM::OFR - 1);  // 16 B multiple
  const unsigned row_bytes = (unsigned)ncopy * (unsigned)sizeof(T);
  const unsigned tx_bytes = row_bytes * SM::NF;

  // zero the exchange and ring memory once (edge threads read never-written slots)
  {
    T* z = reinterpret_cast<T*>(smraw);
    const int nd = (int)(offsetof(SM, bar) / sizeof(T));
    for (int k = t; k < nd; k += NT) z[k] = T(0);
  }
  if (t == 0) {
    for (int s = 0; s < D; ++s) mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {  // load input row rfirst + k into slot k % D
    const int s = k % D;
    const size_t go = off(pitch, x0 - 4, rfirst + k);
    mbar_expect_tx(&sm.bar[s], tx_bytes);
#pragma unroll
    for (int f = 0; f < SM::NF; ++f)
      tma_row(&sm.ring[s][f][SM::OFR], gin[f] + go, row_bytes, &sm.bar[s]);
  };
  if (t == 0) {
    fence_proxy_async();
    for (int k = 0; k < PF && k < niter; ++k) issue(k);
  }

  // ring access: value of field f at iteration-row k, thread column t + dt
#define RG(f, k, dt) sm.ring[(k) % D][f][(t) + SM::OFR + (dt)]
#define XG(a, dt) a[(t) + 1 + (dt)]

  // ---- carried registers (row offsets relative to the newest row L) ----
  // Depth-1 carries are overwritten in place right after their last use, so the
  // register allocator needs no moves for them.
  T vm1 = 0;                 // v(L-1)
  T gam1 = 0, gam2 = 0;      // gamma(L-1), gamma(L-2)
  T PS = 0;                  // K2 y-face force (L-1|L)
  T J0y1 = 0;                // K4 output of row L-1 (the others are read from sm.X2)
  T Hh2 = 0;                 // H_half(L-2)
  T PhS = 0;                 // K5 y-face force (L-3|L-2)
  T phx2h = 0;               // Phi_half_x(L-2)
  T QLx3 = 0, QLy3 = 0;      // Q^L(L-3)
  T ut2 = 0, vt2 = 0, ut3 = 0, vt3 = 0;  // u~, v~ of rows L-2, L-3
  T J0y2 = 0, J0a2 = 0, J0y3 = 0, J0a3 = 0;
  T sy3[4] = {0, 0, 0, 0};   // sigma_y of row L-3 (eta, H, v~, u~)
  T dF3[4] = {0, 0, 0, 0};   // Delta F_x of row L-3
  T Gs[4] = {0, 0, 0, 0};    // y-face flux (L-4|L-3)
  // phase-A results of the newest row, produced at the end of the previous iteration
  T aPE0 = 0, av0 = 0, ar0 = 0, agam0 = 0, aphiy1 = 0;
  bool aw0 = false;
  unsigned long long m0 = 0, m1 = 0, m2 = 0;
  bool neg = false;
  unsigned hist = 0;  // wet flags of rows L..L-4 of this column (bit 0 = row L)
  unsigned wmask = 0;  // HGS band mask of this thread's output cells (see store_update)

  const bool col_out = (t >= 4) && (t < 4 + TX) && (col < nx);
  const bool colg = feeds_xghost(S, col);

  // K8 epilogue for one cell: dry-momentum zeroing, negative-depth flag, stores,
  // wall ghosts and the next step's Eq.7 terms.
  // HGS band mask of this thread's output cells (wet anywhere / in the first or last row
  // of the tile); the first / last column add HGS_LEFT / HGS_RIGHT at the end
  auto store_update = [&](T Hn, T Qxn, T Qyn, T bn, T W3, int j) {
    const bool wet = Hn > Q.eps;
    wmask |= wet ? (HGS_ANY | (j == y0 ? HGS_TOP : 0u) | (j == y1 - 1 ? HGS_BOT : 0u)) : 0u;
    if (!wet) { Qxn = T(0); Qyn = T(0); }
    if (Hn < -Q.neg_tol) neg = true;
    if constexpr (GEN)
      write_with_ghosts(S, oH, oQx, oQy, ob, col, j, Hn, Qxn, Qyn, bn, colg);
    else
      write_wall_ghosts_t(S, oH, oQx, oQy, ob, col, j, Hn, Qxn, Qyn, bn, colg);
    if (wet) {
      T t1, t2, t3;
      dt_terms_t<GEN>(Q, Hn, Qxn, Qyn, W3, aj_at(off(pitch, col, j), Hn),
                    t1, t2, t3);
      unsigned long long a = dbits_t(t1), b = dbits_t(t2), c = dbits_t(t3);
      m0 = a > m0 ? a : m0; m1 = b > m1 ? b : m1; m2 = c > m2 ? c : m2;
    }
  };

  // ================= phase A: K1 + K2 x-face + K2 y-face (row L = rfirst + k) =================
  // Run at the end of the previous iteration, in the same barrier interval as its phase D,
  // so that the long dependency chains of both (K1's 1/H, |v|, H^(-1/3); the x-face HLL)
  // are scheduled together.  Row k's ring slot has been waited for by next_hist().
  auto phaseA = [&](int k) {
    const int L = rfirst + k;
    const int km1 = k - 1 + D;
    const T H0 = RG(F_H, k, 0), b0 = RG(F_B, k, 0);
    const bool w0 = H0 > Q.eps;
    const T eta0 = H0 + b0;
    T r0 = T(0), u0 = T(0), v0 = T(0), gam0 = T(0);
    if (ANYW(w0)) {  // warp-uniform; dry lanes compute on H = 1
      const T Hs = w0 ? H0 : T(1);
      const T rr = rcp_t(Hs);
      const T uu = RG(F_QX, k, 0) * rr, vv = RG(F_QY, k, 0) * rr;
      T gg = T(0);
      if (FRIC) {
        T cgc = Q.cgam;
        if constexpr (GEN) {
          // NEXT-3 field (see fidx: clamped where the result feeds nothing)
          if (S.cg) cgc = S.cg[fidx(col, L)];
        }
        gg = (cgc * sqrt0_t(uu * uu + vv * vv)) * (rr * icbrt_t(Hs));
      }
      r0 = w0 ? rr : T(0); u0 = w0 ? uu : T(0); v0 = w0 ? vv : T(0); gam0 = w0 ? gg : T(0);
    }
    T PE0;
    {
      const T bR = RG(F_B, k, 1);
      PE0 = face_force_t(Q.cPh, eta0, b0, RG(F_H, k, 1) + bR, bR);
    }
    const T H1 = RG(F_H, km1, 0), b1 = RG(F_B, km1, 0);
    const bool w1 = H1 > Q.eps;
    const T PN1 = face_force_t(Q.cPh, H1 + b1, b1, eta0, b0);  // face (L-1|L)
    aphiy1 = w1 ? -(PN1 + PS) : T(0);
    PS = PN1;
    XG(sm.U[k & 1], 0) = u0;
    XG(sm.PE, 0) = PE0;
    aw0 = w0; aPE0 = PE0; av0 = v0; ar0 = r0; agam0 = gam0;
  };

  // The dry decision for iteration k is made at the last barrier of iteration k-1
  // (a __syncthreads_and over "rows L-4..L of my column are dry").
  mbar_wait(&sm.bar[0], 0u);
  hist = RG(F_H, 0, 0) > Q.eps ? 1u : 0u;
  bool cta_dry = __syncthreads_and(hist == 0u);
  if (!cta_dry) phaseA(0);
  int nfull = 0;  // iterations at full cost (this tile's cost for the next step's order)

  constexpr int kUR = (!GEN && sizeof(T) == 8) ? kUnroll : 1;
#pragma unroll kUR
  for (int k = 0; k < niter; ++k) {
    const int L = rfirst + k;  // newest row (strip-local index)
    const int km1 = k - 1 + D, km2 = k - 2 + D, km3 = k - 3 + D;  // non-negative ring rows
    // the slot of row k+PF last held row k+PF-D <= k-5, last read before the previous
    // iteration's barriers
    if (t == 0 && k + PF < niter) {
      fence_proxy_async();
      issue(k + PF);
    }
    auto next_hist = [&]() {
      if (k + 1 < niter) {
        mbar_wait(&sm.bar[(k + 1) % D], (unsigned)(((k + 1) / D) & 1));
        hist = ((hist << 1) | (RG(F_H, k + 1, 0) > Q.eps ? 1u : 0u)) & 31u;
      }
    };
    const int j = L - 3;  // row updated in this iteration
    T Gn[4] = {T(0), T(0), T(0), T(0)};  // (G^H, G^Qx, G^Qy, G^J) at (L-3|L-2)
    T* const X2w = &sm.X2[k & 1][0][0];         // K4 outputs of row L (written in phase D)
    const T* const X2r = &sm.X2[(k - 1) & 1][0][0];  // K4 outputs of row L-1 (read)
#define X2(q, dt) X2r[(q) * SM::XW + (t) + 1 + (dt)]
    if (cta_dry) {
      // Dry fast path (exact): every quantity of R on rows L-4..L is either 0 or the
      // identity, so only the carried window and the row L-3 update run.
      const T H0 = RG(F_H, k, 0);
      gam2 = gam1; gam1 = T(0);
      Hh2 = X2(0, 0);  // row L-1's K4 outputs (exchange row; the previous iteration wrote it)
      phx2h = T(0);
      ut3 = ut2; vt3 = vt2; ut2 = X2(1, 0); vt2 = X2(2, 0);
      J0y3 = J0y2; J0a3 = J0a2; J0y2 = J0y1; J0a2 = X2(4, 0);
      // K4 of the dry row L: H_half = H, u~ = v~ = 0, J0 = 0.  Only H_half goes to the
      // exchange row: this parity's u~, v~, J0 slots hold row L-2's values, which are +0
      // already (rows L-4..L are dry), and a neighbour may still be reading them in the
      // previous iteration's phase D (no barrier in between; racecheck)
      J0y1 = T(0);
      vm1 = T(0);
      X2w[0 * SM::XW + t + 1] = H0;
#pragma unroll
      for (int q = 0; q < 4; ++q) XG(sm.X4[q], 0) = T(0);
      if (col_out && j >= y0 && j < y1) {
        const T H3 = RG(F_H, km3, 0), b3 = RG(F_B, km3, 0);
        const T W3 = HASW ? RG(F_W, km3, 0) : T(S.Wc);
        const T dH = dF3[0] + (Gn[0] - Gs[0]);
        const T dQx = dF3[1] + (Gn[1] - Gs[1]);
        const T dQy = dF3[2] + (Gn[2] - Gs[2]);
        const T dJ = dF3[3] + (Gn[3] - Gs[3]);
        T Hn = fma(-lam, dH, H3);
        T Qxn = fma(-lam, dQx, QLx3);
        T Qyn = fma(-lam, dQy, QLy3);
        const T bn = fma(-(lam * W3), dJ, b3) + (tau * W3) * Q.src;
        if constexpr (GEN) apply_sources(S, tau, off(pitch, col, j), Hn, Qxn, Qyn);
        store_update(Hn, Qxn, Qyn, bn, W3, j);
      }
      QLx3 = T(0); QLy3 = T(0);
#pragma unroll
      for (int q = 0; q < 4; ++q) { dF3[q] = T(0); Gs[q] = T(0); sy3[q] = T(0); }
      next_hist();
      cta_dry = __syncthreads_and(hist == 0u);
      if (!cta_dry && k + 1 < niter) phaseA(k + 1);
      continue;
    }
    ++nfull;
    const T H1 = RG(F_H, km1, 0), b1 = RG(F_B, km1, 0);
    const bool w1 = H1 > Q.eps;
    const T eta1 = H1 + b1;
    __syncthreads();  // ---------------------------------------------------- barrier 1
    {
      // row L-1's K4 outputs: the exchange row written in the previous phase D
      const T Hh1 = X2(0, 0), ut1 = X2(1, 0), vt1 = X2(2, 0), J0a1 = X2(4, 0);
      // ====== phase C: Phi_x (row L), Delta F_x (row L-2), K5 + sigma_x (row L-1),
      //        K6 (row L-2), y-face (L-3|L-2), K8 (row L-3) ======
      const T phix0 = aw0 ? -(aPE0 + XG(sm.PE, -1)) : T(0);

      // Delta F_x of row L-2 from the own face (t|t+1) and the west face (t-1|t)
      T dF2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) dF2[q] = XG(sm.X4[q], 0) - XG(sm.X4[q], -1);
      T PhE1;
      {
        const T bR = RG(F_B, km1, 1);
        PhE1 = face_force_t(Q.cPh, Hh1 + b1, b1, X2(0, 1) + bR, bR);
      }
      T sx1[4];
      {
        const T HLm = RG(F_H, km1, -1), HRp = RG(F_H, km1, 1);
        const T eL = HLm + RG(F_B, km1, -1), eR = HRp + RG(F_B, km1, 1);
        sx1[0] = minmod_t(eta1 - eL, eR - eta1);
        sx1[1] = minmod_t(H1 - HLm, HRp - H1);
        sx1[2] = minmod_t(ut1 - X2(1, -1), X2(1, 1) - ut1);
        sx1[3] = minmod_t(vt1 - X2(2, -1), X2(2, 1) - vt1);
      }
      const T H2 = RG(F_H, km2, 0), b2 = RG(F_B, km2, 0);
      const bool w2 = H2 > Q.eps;
      const T PhN2 = face_force_t(Q.cPh, Hh2 + b2, b2, Hh1 + b1, b1);  // face (L-2|L-1)
      T QLx2 = T(0), QLy2 = T(0);
      if (ANYW(w2)) {
        const T phy2h = -(PhN2 + PhS);
        const T f1 = FRIC ? rcp_t(fma(tau, gam2, T(1))) : T(1);
        const T qx = fma(tau, phx2h, RG(F_QX, km2, 0)) * f1;
        const T qy = fma(tau, phy2h, RG(F_QY, km2, 0)) * f1;
        QLx2 = w2 ? qx : T(0); QLy2 = w2 ? qy : T(0);
      }
      PhS = PhN2;
      Hh2 = Hh1;
      // y-face (L-3|L-2): sigma_y of row L-2 (always: it is carried), HLL, sediment
      const T H3 = RG(F_H, km3, 0), b3 = RG(F_B, km3, 0);
      const bool w3 = H3 > Q.eps;
      const T eta2 = H2 + b2, eta3 = H3 + b3;
      T sy2[4];
      sy2[0] = minmod_t(eta2 - eta3, eta1 - eta2);
      sy2[1] = minmod_t(H2 - H3, H1 - H2);
      sy2[2] = minmod_t(vt2 - vt3, vt1 - vt2);
      sy2[3] = minmod_t(ut2 - ut3, ut1 - ut2);
      if (ANYW(w3 || w2)) {
        const bool any = w3 || w2;
        hll_bf(Q.g, fma(T(0.5), sy3[0], eta3), fma(T(0.5), sy3[1], H3), fma(T(0.5), sy3[2], vt3),
                 fma(T(0.5), sy3[3], ut3), fma(T(-0.5), sy2[0], eta2), fma(T(-0.5), sy2[1], H2),
                 fma(T(-0.5), sy2[2], vt2), fma(T(-0.5), sy2[3], ut2), !any,
                 Gn[0], Gn[2], Gn[1]);  // normal momentum of a y-face -> Qy, tangential -> Qx
        Gn[3] = (any && TRANSP) ? sed_face_t(Q, vt3, vt2, J0y3, J0y2, J0a3, J0a2, b3, b2)
                                     : T(0);
      }
      ut3 = ut2; vt3 = vt2; ut2 = ut1; vt2 = vt1;
      J0y3 = J0y2; J0a3 = J0a2; J0y2 = J0y1; J0a2 = J0a1;
#pragma unroll
      for (int q = 0; q < 4; ++q) sy3[q] = sy2[q];
      // ---- K8 update of row L-3 (its last input, the y-face (L-3|L-2), is ready) ----
      if (col_out && j >= y0 && j < y1) {
        const T W3 = HASW ? RG(F_W, km3, 0) : T(S.Wc);
        const T dH = dF3[0] + (Gn[0] - Gs[0]);
        const T dQx = dF3[1] + (Gn[1] - Gs[1]);
        const T dQy = dF3[2] + (Gn[2] - Gs[2]);
        const T dJ = dF3[3] + (Gn[3] - Gs[3]);
        T Hn = fma(-lam, dH, H3);
        T Qxn = fma(-lam, dQx, QLx3);
        T Qyn = fma(-lam, dQy, QLy3);
        const T bn = fma(-(lam * W3), dJ, b3) + (tau * W3) * Q.src;
        if constexpr (GEN) apply_sources(S, tau, off(pitch, col, j), Hn, Qxn, Qyn);
        store_update(Hn, Qxn, Qyn, bn, W3, j);
      }
      QLx3 = QLx2; QLy3 = QLy2;
#pragma unroll
      for (int q = 0; q < 4; ++q) { dF3[q] = dF2[q]; Gs[q] = Gn[q]; }
      XG(sm.X3[0], 0) = PhE1;
#pragma unroll
      for (int q = 0; q < 4; ++q) XG(sm.X3[1 + q], 0) = sx1[q];
      next_hist();
      const bool dry_next = __syncthreads_and(hist == 0u);  // ---------------- barrier 2
      // ====== phase D: Phi_half_x + x-face flux (row L-1), phase A (row L+1), K4 + J0
      //        (row L) ======
      phx2h = w1 ? -(XG(sm.X3[0], 0) + XG(sm.X3[0], -1)) : T(0);
      T Fn[4] = {T(0), T(0), T(0), T(0)};
      {
        // own-side values of row L-1 re-read (exchange rows, ring) instead of carried
        const T H1 = RG(F_H, km1, 0), b1 = RG(F_B, km1, 0);
        const T eta1 = H1 + b1;
        const T ut1 = X2(1, 0), vt1 = X2(2, 0), J0x1 = X2(3, 0), J0a1 = X2(4, 0);
        const T HR = RG(F_H, km1, 1);
        const bool any = (gt_u(H1, Q.eps) | gt_u(HR, Q.eps)) != 0u;
        if (ANYW(any)) {
          const T bR = RG(F_B, km1, 1);
          const T eR = HR + bR;
          const T uR = X2(1, 1), vR = X2(2, 1);
          // own slopes sigma_x of row L-1: the exchange row written in phase C
          hll_bf(Q.g, fma(T(0.5), XG(sm.X3[1], 0), eta1), fma(T(0.5), XG(sm.X3[2], 0), H1),
                   fma(T(0.5), XG(sm.X3[3], 0), ut1), fma(T(0.5), XG(sm.X3[4], 0), vt1),
                   fma(T(-0.5), XG(sm.X3[1], 1), eR), fma(T(-0.5), XG(sm.X3[2], 1), HR),
                   fma(T(-0.5), XG(sm.X3[3], 1), uR), fma(T(-0.5), XG(sm.X3[4], 1), vR), !any,
                   Fn[0], Fn[1], Fn[2]);  // normal momentum of an x-face -> Qx, tangential -> Qy
          Fn[3] = (any && TRANSP) ? sed_face_t(Q, ut1, uR, J0x1, X2(3, 1), J0a1, X2(4, 1), b1, bR)
                                       : T(0);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) XG(sm.X4[q], 0) = Fn[q];
      // phase A of the next row, unconditionally (a wasted row at a wet -> dry change;
      // beyond the last row it reads a stale but finite ring slot and feeds nothing);
      // the row-L values it replaces are kept for K4
      const bool w0 = aw0;
      const T r0 = ar0, gam0 = agam0, v0 = av0;
      phaseA(k + 1);
      // ---- K4 predictor + J0 of row L (its x-neighbours' u and Phi_x: barrier 1) ----
      {
        const T H0 = RG(F_H, k, 0);
        T Hh = H0, ut = T(0), vt = T(0);
        if (ANYW(w0)) {
          const T* Uc = sm.U[k & 1];
          T div = ((XG(Uc, 1) - XG(Uc, -1)) + (av0 - vm1)) * Q.inv_2h;
          const T hh = H0 * fma(-theta, div, T(1));
          const T f = FRIC ? rcp_t(fma(theta, gam0, T(1))) : T(1);  // gam0 = 0 when dry
          const T uu = (fma(theta, phix0, RG(F_QX, k, 0)) * f) * r0;
          const T vv = (fma(theta, aphiy1, RG(F_QY, k, 0)) * f) * r0;
          Hh = w0 ? hh : H0; ut = w0 ? uu : T(0); vt = w0 ? vv : T(0);
        }
        T jx = T(0), jy = T(0), ja = T(0);
        if (TRANSP) grass_t<GEN>(Q, ut, vt, H0, aj_at(fidx(col, L), H0), jx, jy, ja);
        X2w[0 * SM::XW + t + 1] = Hh;
        X2w[1 * SM::XW + t + 1] = ut;
        X2w[2 * SM::XW + t + 1] = vt;
        X2w[3 * SM::XW + t + 1] = jx;
        X2w[4 * SM::XW + t + 1] = ja;
        J0y1 = jy;
        vm1 = v0;
        gam2 = gam1; gam1 = gam0;
      }
      cta_dry = dry_next;
    }
#undef X2
  }
#undef RG
#undef XG
  // negative depth (reading #27): a 4th max slot, combined across strips and ranks with the
  // Eq.7 maxima, so every strip stops at the same step
  if (neg) atomicMax(&gM[3], 1ull);
  // block max of the Eq.7 terms, one atomicMax per CTA and term
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, m0, o);
    unsigned long long b = __shfl_xor_sync(0xffffffffu, m1, o);
    unsigned long long c = __shfl_xor_sync(0xffffffffu, m2, o);
    m0 = a > m0 ? a : m0; m1 = b > m1 ? b : m1; m2 = c > m2 ? c : m2;
  }
  if ((t & 31) == 0) {
    sm.red[0][t >> 5] = m0; sm.red[1][t >> 5] = m1; sm.red[2][t >> 5] = m2;
  }
  {
    const int xe = min(x0 + TX, nx);  // the tile's last column + 1
    if (wmask & HGS_ANY) wmask |= (col == x0 ? HGS_LEFT : 0u) | (col == xe - 1 ? HGS_RIGHT : 0u);
  }
  wmask = __reduce_or_sync(0xffffffffu, wmask);
  if ((t & 31) == 0) sm.wm[t >> 5] = wmask;
  __syncthreads();
  if (t == 0 && hg.enable) {
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) m |= sm.wm[w];
    hg.fnext[ti] = (unsigned char)m;
    hg.tstate[ti] = 0;
    push_flags(m);
  }
  push_rows();  // after the barrier above: every thread's rows are written
  if (t == 0 && hg.cost) hg.cost[ti] = (unsigned short)min(nfull, 65535);
  if (t == 0 && hg.stats) atomicAdd(&hg.stats[0], 1ull);
  if (t < 3) {
    unsigned long long m = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) m = sm.red[t][w] > m ? sm.red[t][w] : m;
    if (m) atomicMax(&gM[t], m);
  }
}

template <typename T, int NT, bool HASW, int D, int PF, int MINB, bool GEN>
void launch_t(const StripView& S, Ctrl* C, const Phys& P, unsigned long long* gM, int row0,
              int row1, int TY, const Hgs& hg, cudaStream_t st) {
  using SM = Smem<T, NT, HASW, D>;
  constexpr int TX = NT - 8;
  // the dynamic shared-memory limit is a per-device attribute: set it once per device (a
  // failure leaves the bit clear and surfaces as the launch error the caller checks)
  static unsigned long long configured = 0;
  const size_t smem = sizeof(SM);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((configured >> (dev & 63)) & 1ull)) {
    if (cudaFuncSetAttribute(fused_step_kernel<T, NT, HASW, D, PF, MINB, GEN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess)
      configured |= 1ull << (dev & 63);
  }
  // one-dimensional: CTA i marches tile hg.order[i] (or i), tile (bx, by) = (i % gx, i / gx)
  dim3 grid((unsigned)((S.nx + TX - 1) / TX) * (unsigned)((row1 - row0 + TY - 1) / TY));
  fused_step_kernel<T, NT, HASW, D, PF, MINB, GEN>
      <<<grid, NT, smem, st>>>(S, C, P, gM, row0, row1, TY, hg);
}

template <int NT, int D, int PF, int MINB>
void launch_v(const StripView& S, Ctrl* C, const Phys& P, unsigned long long* gM, int row0,
              int row1, int TY, const Hgs& hg, cudaStream_t st) {
  Hgs h = hg;
  if (NT - 8 != FUSED_TX) h.enable = 0;  // tiling of the flags is FUSED_TX wide
  if (S.prec == 4) {  // NEXT-2 fp32 mode: hot-path features only (checked at create)
    // fp32 state halves the ring and the registers: one more resident CTA per SM
    if (S.W) launch_t<float, NT, true, D, PF, kMinB32, false>(S, C, P, gM, row0, row1, TY, h, st);
    else launch_t<float, NT, false, D, PF, kMinB32, false>(S, C, P, gM, row0, row1, TY, h, st);
    return;
  }
  // GEN: NEXT-3/4 features present or a physics term switched off; otherwise the
  // hot-path specialisation
  const bool gen = !P.fric || !P.transport || P.m_grass != 2 || P.m_real >= 0.0 || P.aj_mode || S.cg || S.beta || S.aj0 || S.bc_xlo != 1 ||
                   S.bc_xhi != 1 || S.wall_lo == 2 || S.wall_hi == 2 ||
                   !(P.g * P.eps >= 0x1p-890);  // dt_terms: sqrt(g H) without the zero guard
  if (S.W) {
    if (gen) launch_t<double, NT, true, D, PF, MINB, true>(S, C, P, gM, row0, row1, TY, h, st);
    else launch_t<double, NT, true, D, PF, MINB, false>(S, C, P, gM, row0, row1, TY, h, st);
  } else {
    if (gen) launch_t<double, NT, false, D, PF, MINB, true>(S, C, P, gM, row0, row1, TY, h, st);
    else launch_t<double, NT, false, D, PF, MINB, false>(S, C, P, gM, row0, row1, TY, h, st);
  }
}

// Counting sort of a launch's tiles by descending cost: one CTA.  Each
// thread loads its keys for a chunk of kOrdChunk tiles at once (one memory latency per
// chunk, not one per key) and keeps them for the scatter; the shared-memory atomics are
// warp-aggregated (most tiles share the key of cost 0).
constexpr int kOrdBuckets = 256;
constexpr int kOrdThreads = 1024;
constexpr int kOrdPer = 24;  // keys per thread per chunk
constexpr int kOrdChunk = kOrdThreads * kOrdPer;
__global__ void __launch_bounds__(kOrdThreads, 1) order_tiles_kernel(
    const unsigned short* __restrict__ cost, int ntx, int tr0, int tr1, int* __restrict__ order) {
  __shared__ int cnt[kOrdBuckets];
  __shared__ int wsum[kOrdBuckets / 32];
  const int n = ntx * (tr1 - tr0);
  const int t = threadIdx.x, lane = t & 31;
  const unsigned short* c = cost + (size_t)tr0 * ntx;
  auto key_of = [&](int i) { return kOrdBuckets - 1 - min((int)__ldg(c + i), kOrdBuckets - 1); };
  // warp-aggregated atomicAdd of 1 per lane on cnt[key]; returns this lane's old value
  auto agg_add = [&](unsigned act, int key) {
    // a warp whose keys are all equal (common: runs of dry tiles) skips the match
    const unsigned m = __all_sync(act, key == __shfl_sync(act, key, __ffs(act) - 1))
                           ? act : __match_any_sync(act, key);
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cnt[key], __popc(m));
    return __shfl_sync(m, base, leader) + __popc(m & ((1u << lane) - 1u));
  };
  for (int b = t; b < kOrdBuckets; b += kOrdThreads) cnt[b] = 0;
  __syncthreads();
  int key[kOrdPer];
  for (int c0 = 0; c0 < n; c0 += kOrdChunk) {  // pass 1: histogram (bucket 0 = costliest)
#pragma unroll
    for (int q = 0; q < kOrdPer; ++q) {
      const int i = c0 + q * kOrdThreads + t;
      key[q] = i < n ? key_of(i) : -1;
    }
#pragma unroll
    for (int q = 0; q < kOrdPer; ++q) {
      const unsigned act = __ballot_sync(0xffffffffu, key[q] >= 0);
      if (key[q] >= 0) agg_add(act, key[q]);
    }
  }
  __syncthreads();
  int x = 0, incl = 0;  // exclusive scan of the 256 counts: 8 warps, then the warp totals
  if (t < kOrdBuckets) {
    x = cnt[t];
    incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[t >> 5] = incl;
  }
  __syncthreads();
  if (t < kOrdBuckets) {
    int base = 0;
    for (int w = 0; w < (t >> 5); ++w) base += wsum[w];
    cnt[t] = base + incl - x;
  }
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += kOrdChunk) {  // pass 2: scatter (keys still held when n fits)
    if (n > kOrdChunk) {
#pragma unroll
      for (int q = 0; q < kOrdPer; ++q) {
        const int i = c0 + q * kOrdThreads + t;
        key[q] = i < n ? key_of(i) : -1;
      }
    }
#pragma unroll
    for (int q = 0; q < kOrdPer; ++q) {
      const unsigned act = __ballot_sync(0xffffffffu, key[q] >= 0);
      if (key[q] >= 0) order[agg_add(act, key[q])] = c0 + q * kOrdThreads + t;
    }
  }
}

__global__ void order_identity_kernel(int* order, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) order[i] = i;
}

}  // namespace

void launch_order_identity(int* order, int n, cudaStream_t st, long long* nlaunch) {
  if (n <= 0) return;
  order_identity_kernel<<<(n + 255) / 256, 256, 0, st>>>(order, n);
  *nlaunch += 1;
}

void launch_order_tiles(const unsigned short* cost, int ntx, int tr0, int tr1, int* order,
                        cudaStream_t st, long long* nlaunch) {
  if (tr1 <= tr0) return;
  order_tiles_kernel<<<1, kOrdThreads, 0, st>>>(cost, ntx, tr0, tr1, order);
  *nlaunch += 1;
}

void launch_fused_step(const StripView& S, Ctrl* C, const Phys& P, unsigned long long* gM,
                       int row0, int row1, int tile_rows, const Hgs& hg, cudaStream_t st,
                       long long* nlaunch) {
  if (row1 <= row0) return;
  const int TY = tile_rows > 0 ? tile_rows : 128;
  // 128 threads (120 output columns), an 8-row TMA ring prefetching 3 rows ahead,
  // 3 resident CTAs per SM in fp64 (5 in fp32: <= 102 registers, 89 used, no spills)
#ifndef CSPH_RING
#define CSPH_RING 8   // development knobs: ring slots, prefetch distance
#define CSPH_PF 3
#endif
  launch_v<FUSED_NT, CSPH_RING, CSPH_PF, FUSED_MINB>(S, C, P, gM, row0, row1, TY, hg, st);
  *nlaunch += 1;
}

}  // namespace ck
