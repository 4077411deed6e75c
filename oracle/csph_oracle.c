/*
 * csph_oracle.c -- TEST INFRASTRUCTURE ONLY (see csph_oracle.h).
 *
 * A plain, slow, single-threaded implementation of one CSPH-TVD step in the
 * reading R of DESIGN.md section 3.  Every stage of R is its own loop nest
 * over the grid with its intermediates materialised, in the paper's kernel
 * order K1..K8.  No blocking, fusion or reordering.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 * (IEEE binary64, round-to-nearest, no implicit FMA contraction).
 *
 * The same source built with -DORC_FP32 is R evaluated in IEEE binary32 (DESIGN.md 3.14,
 * the NEXT-2 fp32 mode): state, intermediates and every per-cell operation in float, so
 * every decision of R (wet test, gate, donor, HLL case, minmod) is taken in the precision
 * the fp32 mode computes in; host constants are computed in double and rounded once to
 * float; tau is computed in double from the float maxima widened exactly (Eq.7 on the
 * host side of the step), then rounded to float for the step.  x^(-1/3) in fp32 is the
 * pinned binary32 recipe of DESIGN.md 3.14.  Public entry points keep double arguments.
 */
#include "csph_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef ORC_FP32
typedef float real;
#define SQRT sqrtf
#define FMA fmaf
#else
typedef double real;
#define SQRT sqrt
#define FMA fma
#endif
#define RL(x) ((real)(x))  /* a constant of R in the working precision */

#define G 3 /* ghost layers: the stencil radius of R */

struct orc {
  int nx, ny, pw, ph; /* interior size, padded width/height */
  double h;           /* cell size ("h is cell size") */
  orc_params p;
  /* host-side constants of R, computed in double, then rounded once to
   * the working precision */
  real inv_h, inv_2h, cPh, cgam, kappa;
  real hbm;  /* reading #31 cut-off depth: h_bed_min, or d50 when h_bed_min < 0 */
  real eps, neg_tol, g, A_J, C_J, C_Sh, d50, s_rel, src;
  int wall[4];
  int have_state;
  /* state U = (H, Hu, Hv, b) of Eq.6 and W = 1/(1-psi) of Eq.1 */
  real *H, *Qx, *Qy, *b, *W;
  /* intermediates (padded) */
  real *eta, *r, *u, *v, *phix, *phiy, *gam, *Hh, *ut, *vt, *phix2, *phiy2;
  real *QLx, *QLy, *J0x, *J0y, *J0a;
  real *FH, *FQx, *FQy, *FJ, *GH, *GQx, *GQy, *GJ;
  real *Hn, *Qxn, *Qyn, *bn;
  /* NEXT-3 spatial inputs (P:129 n_M(x,y), beta(x,y); Eq.6 sigma):
   * per-cell c_gam = g n_M^2, absorption beta and source s (rain + point inflow) */
  real *cg, *beta, *srcf, *nfld;
  int has_fields, fields_fric, fields_src;
  unsigned char* w;
  double M[3];
  double t, last_dt;
  long long steps;
};

#define IDX(o, i, j) ((size_t)((j) + G) * (size_t)(o)->pw + (size_t)((i) + G))

/* ---- small pieces of R (in the working precision `real`) ------------------ */

/* explicit selects, never fmin/fmax */
static real sel_min(real a, real b) { return (a < b) ? a : b; }
static real sel_max(real a, real b) { return (a > b) ? a : b; }

/* minmod TVD limiter ("TVD-limiters"; reading #12) */
static real r_minmod(real a, real b) {
  if (a > RL(0) && b > RL(0)) return sel_min(a, b);
  if (a < RL(0) && b < RL(0)) return sel_max(a, b);
  return RL(0);
}

#ifdef ORC_FP32
/* pinned binary32 x^(-1/3) for x > 0 normal: integer seed from the bits,
 * then 3 Newton steps y <- y + y*((1 - x*y^3)*(1/3)) */
static real r_icbrt(real x) {
  int32_t bits;
  memcpy(&bits, &x, 4);
  int32_t yb = 0x54A2FA8C - bits / 3;
  real y;
  memcpy(&y, &yb, 4);
  const real third = RL(1) / RL(3);
  for (int k = 0; k < 3; ++k) y = FMA(y, FMA(-x, (y * y) * y, RL(1)) * third, y);
  return y;
}
#else
/* pinned x^(-1/3) for x > 0 normal: integer seed from the
 * exponent bits, then 5 Newton steps y <- y + y*((1 - x*y^3)*(1/3)). */
static real r_icbrt(real x) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  uint64_t yb = 0x553F751EB851EC00ull - bits / 3ull;
  real y;
  memcpy(&y, &yb, 8);
  const real third = 1.0 / 3.0;
  for (int k = 0; k < 5; ++k) {
    real y3 = (y * y) * y;
    real e = FMA(-x, y3, 1.0) * third;
    y = FMA(y, e, y);
  }
  return y;
}
#endif

/* Pinned x^q for x >= 0, q >= 0 (NEXT-4 real Grass exponent): IEEE + - x /
 * and integer bit operations only, the same sequence on CPU and GPU, so both sides agree
 * bitwise; not correctly rounded (pinned vs 50-digit mpmath, <= 1e-13 relative).
 *   x^0 = 1, 0^q = 0 (q > 0);  x = f 2^e with f in [sqrt(1/2), sqrt(2));
 *   ln f = 2 atanh(z) = 2 z (1 + z^2/3 + ... + z^22/23), z = (f-1)/(f+1), |z| <= 0.1716;
 *   y = q e + (q ln f) / ln 2 = q log2 x;  y < -1021 -> 0, y > 1023 -> +inf;
 *   n = nearest integer to y (the 1.5 2^52 trick), r = y - n in [-1/2, 1/2] (exact);
 *   2^r = exp(r ln 2) by its Taylor series to degree 14;  x^q = 2^r 2^n. */
static double pow_pinned(double x, double q) {
  static const double A[12] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                               0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                               0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                               0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
  static const double E[15] = {0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1,
                               0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
                               0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,
                               0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
                               0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37};
  if (q == 0.0) return 1.0;
  if (!(x > 0.0)) return 0.0;
  uint64_t bits;
  memcpy(&bits, &x, 8);
  int e = (int)((bits >> 52) & 0x7FF);
  if (e == 0) {  /* subnormal: scale by 2^64 (exact) */
    double xs = x * 0x1p64;
    memcpy(&bits, &xs, 8);
    e = (int)((bits >> 52) & 0x7FF) - 64;
  }
  e -= 1023;
  uint64_t fb = (bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  double f;
  memcpy(&f, &fb, 8);
  if (f > 0x1.6a09e667f3bcdp+0) { f = 0.5 * f; e += 1; }
  double z = (f - 1.0) / (f + 1.0);
  double w = z * z;
  double p = A[11];
  for (int k = 10; k >= 0; --k) p = p * w + A[k];
  double lnf = (2.0 * z) * p;
  double y = q * (double)e + (q * lnf) * 0x1.71547652b82fep+0;
  if (y < -1021.0) return 0.0;
  if (y > 1023.0) return INFINITY;
  double n = (y + 0x1.8p52) - 0x1.8p52;
  double r = y - n;
  double t = r * 0x1.62e42fefa39efp-1;
  double s = E[14];
  for (int k = 13; k >= 0; --k) s = s * t + E[k];
  uint64_t sb = (uint64_t)((int64_t)n + 1023) << 52;
  double sc;
  memcpy(&sc, &sb, 8);
  return s * sc;
}

double orc_pow_pinned(double x, double q) { return pow_pinned(x, q); }

/* Eq.3 with integer m (m = 2 on the hot path, NEXT-4 any 0..8): p = |v|^m by
 * repeated multiplication in s2 = |v|^2, then J0 = (A p) v and |J0| = (A p) |v|.  For
 * m = 2: p = 1 * s2 = s2 exactly, i.e. J0 = A_J v |v|^2, |J0| = A_J |v|^3.  A real
 * exponent mr >= 0 (NEXT-4, m_real) takes p = pow_pinned(s2, mr/2) instead. */
static real grass_pow(int m, double mr, real s2, real a) {
  if (mr >= 0.0) return RL(pow_pinned((double)s2, 0.5 * mr));
  real pw = RL(1);
  for (int k = 0; k < m / 2; ++k) pw = pw * s2;
  if (m % 2) pw = pw * a;
  return pw;
}

static void r_grass_mr(real A, int m, double mr, real vx, real vy, real* jx, real* jy, real* jabs) {
  real s2 = vx * vx + vy * vy;
  real a = SQRT(s2);
  real pw = grass_pow(m, mr, s2, a);
  real c = A * pw;
  *jx = c * vx;
  *jy = c * vy;
  *jabs = c * a;
}

/* Eq.4, A_J from the local depth H (reading #5: H = local depth) */
static real r_aj_eq4(real g, real n_manning, real s_rel, real H, real d50) {
  return (RL(0.05) * ((n_manning * n_manning) * n_manning)) / (((s_rel - RL(1)) * SQRT(g * H)) * d50);
}

/* Eq.2, vector reading #4: J_n = J0_n - C_J |J0| db/dn */
static real r_slope_flux(real J0n, real J0abs, real C_J, real db_dn) {
  return FMA(-(C_J * J0abs), db_dn, J0n);
}

/* Eq.5 Shamov gate, reading #6: |v| > v_k  <=>  s2^3 > kappa*H */
static int r_shamov_gate(real kappa, real s2, real H, real C_Sh) {
  if (C_Sh == RL(0)) return 1;
  return ((s2 * s2) * s2 > kappa * H) ? 1 : 0;
}

/* Reading #31: bedload needs a water column deeper than h_bed_min, by default the grain
 * size d50 -- no transport where H <= h_bed_min (Eq.5's critical velocity C_Sh d50^(1/3)
 * H^(1/6) vanishes as H -> 0, so the gate alone would let films thinner than a grain carry
 * sediment).  h_bed_min = 0 is the literal Eq.5. */
static int r_bed_mobile(real H, real h_bed_min) {
  return H > h_bed_min ? 1 : 0;
}

/* Face pressure term of K2/K5 (Eq.6 row 2, -gH grad(H+b), reading #1;
 * DESIGN.md 3.3) in hydrostatic-reconstruction form:
 *   b* = max(b_L, b_R) (cell beds), H*_s = max(0, eta_s - b*),
 *   P  = (c_P/2 * (H*_L + H*_R)) * (H*_R - H*_L),  c_P/2 = g/(4h) a host constant
 * (= c_P * (0.5*(H*_L + H*_R)) exactly unless the sum is subnormal).
 * The wet flags are not needed: a dry cell whose bed is above the water has
 * H* = 0 on both sides of the face (a wall), a lower dry cell drives the flow. */
static real face_force(real cPh, real etaL, real bL, real etaR, real bR) {
  real bs = sel_max(bL, bR);
  real HsL = sel_max(RL(0), etaL - bs);
  real HsR = sel_max(RL(0), etaR - bs);
  return (cPh * (HsL + HsR)) * (HsR - HsL);
}

/* K7: hydrostatic step + HLL on F = (Hu, Hu^2, Huv) (Eq.6) */
static void r_hll_face(real g, real eta_m, real H_m, real un_m, real ut_m,
                       real eta_p, real H_p, real un_p, real ut_p,
                       int wL, int wR, real out[3]) {
  out[0] = RL(0); out[1] = RL(0); out[2] = RL(0);
  if (!wL && !wR) return;
  real b_m = eta_m - H_m, b_p = eta_p - H_p;
  real bs = sel_max(b_m, b_p);
  real Hs_m = sel_max(RL(0), eta_m - bs);
  real Hs_p = sel_max(RL(0), eta_p - bs);
  int dry_m = !(Hs_m > RL(0)), dry_p = !(Hs_p > RL(0));
  if (dry_m && dry_p) return;
  real m_m = Hs_m * un_m, m_p = Hs_p * un_p;
  real FL[3] = {m_m, m_m * un_m, m_m * ut_m};
  real FR[3] = {m_p, m_p * un_p, m_p * ut_p};
  real UL[3] = {Hs_m, m_m, Hs_m * ut_m};
  real UR[3] = {Hs_p, m_p, Hs_p * ut_p};
  real SL, SR;
  if (!dry_m && !dry_p) {
    real c_m = SQRT(g * Hs_m), c_p = SQRT(g * Hs_p);
    SL = sel_min(un_m - c_m, un_p - c_p);
    SR = sel_max(un_m + c_m, un_p + c_p);
  } else if (dry_p) {
    real c_m = SQRT(g * Hs_m);
    SL = un_m - c_m;
    SR = un_m + RL(2) * c_m;
  } else {
    real c_p = SQRT(g * Hs_p);
    SL = un_p - RL(2) * c_p;
    SR = un_p + c_p;
  }
  if (SL >= RL(0)) {
    for (int k = 0; k < 3; ++k) out[k] = FL[k];
  } else if (SR <= RL(0)) {
    for (int k = 0; k < 3; ++k) out[k] = FR[k];
  } else {
    real inv = RL(1) / (SR - SL);
    real SLSR = SL * SR;
    for (int k = 0; k < 3; ++k)
      out[k] = ((SR * FL[k] - SL * FR[k]) + SLSR * (UR[k] - UL[k])) * inv;
  }
}

/* ---- public double entry points of the pieces (pins) ---------------------- */

double orc_minmod(double a, double b) { return r_minmod(RL(a), RL(b)); }
double orc_icbrt(double x) { return r_icbrt(RL(x)); }

void orc_grass(double A_J, double vx, double vy, double* jx, double* jy, double* jabs) {
  orc_grass_m(A_J, 2, vx, vy, jx, jy, jabs);
}

void orc_grass_m(double A, int m, double vx, double vy, double* jx, double* jy, double* jabs) {
  real x, y, a;
  r_grass_mr(RL(A), m, -1.0, RL(vx), RL(vy), &x, &y, &a);
  *jx = x; *jy = y; *jabs = a;
}

double orc_aj_eq4(double g, double n_manning, double s_rel, double H, double d50) {
  return r_aj_eq4(RL(g), RL(n_manning), RL(s_rel), RL(H), RL(d50));
}

double orc_slope_flux(double J0n, double J0abs, double C_J, double db_dn) {
  return r_slope_flux(RL(J0n), RL(J0abs), RL(C_J), RL(db_dn));
}

int orc_shamov_gate(double kappa, double s2, double H, double C_Sh) {
  return r_shamov_gate(RL(kappa), RL(s2), RL(H), RL(C_Sh));
}

int orc_bed_mobile(double H, double h_bed_min) { return r_bed_mobile(RL(H), RL(h_bed_min)); }

/* Manning friction coefficient (reading #19): gamma = g n^2 |v| / H^(4/3),
 * written as (c_gam*s)*(r*H^(-1/3)) with r = 1/H. */
double orc_gamma(const orc_params* p, double H, double u, double v) {
  if (!(p->n_manning > 0.0)) return 0.0;
  real cg = RL(p->g * (p->n_manning * p->n_manning));
  real uu = RL(u), vv = RL(v), Hh = RL(H);
  real s = SQRT(uu * uu + vv * vv);
  real r = RL(1) / Hh;
  return (cg * s) * (r * r_icbrt(Hh));
}

void orc_hll_face(double g, double eta_m, double H_m, double un_m, double ut_m,
                  double eta_p, double H_p, double un_p, double ut_p,
                  int wL, int wR, double out[3]) {
  real o[3];
  r_hll_face(RL(g), RL(eta_m), RL(H_m), RL(un_m), RL(ut_m), RL(eta_p), RL(H_p), RL(un_p),
             RL(ut_p), wL, wR, o);
  for (int k = 0; k < 3; ++k) out[k] = o[k];
}

/* ---- lifecycle ------------------------------------------------------------ */

static int valid_params(const orc_params* p) {
  if (!(p->g > 0.0) || !isfinite(p->g)) return 0;
  if (!(p->K > 0.0 && p->K < 1.0)) return 0;
  if (!(p->eps_dry >= 0.0) || !isfinite(p->eps_dry)) return 0;
  if (!(p->dt_max > 0.0)) return 0;
  if (!(p->neg_tol >= 0.0)) return 0;
  if (!(p->n_manning >= 0.0) || !isfinite(p->n_manning)) return 0;
  if (!(p->A_J >= 0.0) || !isfinite(p->A_J)) return 0;
  if (p->m_grass < 0 || p->m_grass > 8) return 0;
  if (p->aj_mode != 0 && p->aj_mode != 1) return 0;
  if (p->aj_mode == 1 && !(p->s_rel > 1.0 && isfinite(p->s_rel) && p->d50 > 0.0)) return 0;
  if (!isfinite(p->C_J)) return 0;
  if (!(p->C_Sh >= 0.0) || !isfinite(p->C_Sh)) return 0;
  if (p->C_Sh > 0.0 && !(p->d50 > 0.0)) return 0;
  if (!isfinite(p->q_plus) || !isfinite(p->q_minus)) return 0;
  if (!isfinite(p->h_bed_min)) return 0;
  if (!(p->m_real < 0.0) && !(p->m_real >= 0.0 && p->m_real <= 8.0)) return 0;
  return 1;
}

orc_t* orc_create(int nx, int ny, double dx, const orc_params* p) {
  if (nx < 3 || ny < 3 || !(dx > 0.0) || !isfinite(dx) || !p || !valid_params(p)) return NULL;
  orc_t* o = (orc_t*)calloc(1, sizeof(orc_t));
  if (!o) return NULL;
  o->nx = nx; o->ny = ny; o->pw = nx + 2 * G; o->ph = ny + 2 * G;
  o->h = dx; o->p = *p;
  o->inv_h = RL(1.0 / dx);
  o->inv_2h = RL(1.0 / (2.0 * dx));
  o->cPh = RL(0.5 * (p->g / (2.0 * dx)));  /* c_P/2 = g/(4h) */
  o->cgam = RL(p->g * (p->n_manning * p->n_manning));
  {
    double c2 = p->C_Sh * p->C_Sh;
    o->kappa = RL(((c2 * c2) * c2) * (p->d50 * p->d50));
  }
  o->hbm = RL(p->h_bed_min < 0.0 ? p->d50 : p->h_bed_min);
  o->eps = RL(p->eps_dry); o->neg_tol = RL(p->neg_tol); o->g = RL(p->g);
  o->A_J = RL(p->A_J); o->C_J = RL(p->C_J); o->C_Sh = RL(p->C_Sh); o->d50 = RL(p->d50);
  o->s_rel = RL(p->s_rel); o->src = RL(p->q_plus - p->q_minus);
  for (int s = 0; s < 4; ++s) o->wall[s] = 1;
  size_t n = (size_t)o->pw * (size_t)o->ph;
  real** arrs[] = {&o->H, &o->Qx, &o->Qy, &o->b, &o->W, &o->eta, &o->r, &o->u, &o->v,
                     &o->phix, &o->phiy, &o->gam, &o->Hh, &o->ut, &o->vt, &o->phix2,
                     &o->phiy2, &o->QLx, &o->QLy, &o->J0x, &o->J0y, &o->J0a, &o->FH,
                     &o->FQx, &o->FQy, &o->FJ, &o->GH, &o->GQx, &o->GQy, &o->GJ,
                     &o->Hn, &o->Qxn, &o->Qyn, &o->bn, &o->cg, &o->beta, &o->srcf, &o->nfld};
  for (size_t k = 0; k < sizeof(arrs) / sizeof(arrs[0]); ++k) {
    *arrs[k] = (real*)calloc(n, sizeof(real));
    if (!*arrs[k]) { orc_destroy(o); return NULL; }
  }
  o->w = (unsigned char*)calloc(n, 1);
  if (!o->w) { orc_destroy(o); return NULL; }
  return o;
}

void orc_destroy(orc_t* o) {
  if (!o) return;
  real* arrs[] = {o->H, o->Qx, o->Qy, o->b, o->W, o->eta, o->r, o->u, o->v, o->phix,
                    o->phiy, o->gam, o->Hh, o->ut, o->vt, o->phix2, o->phiy2, o->QLx,
                    o->QLy, o->J0x, o->J0y, o->J0a, o->FH, o->FQx, o->FQy, o->FJ,
                    o->GH, o->GQx, o->GQy, o->GJ, o->Hn, o->Qxn, o->Qyn, o->bn,
                    o->cg, o->beta, o->srcf, o->nfld};
  for (size_t k = 0; k < sizeof(arrs) / sizeof(arrs[0]); ++k) free(arrs[k]);
  free(o->w);
  free(o);
}

int orc_set_walls(orc_t* o, int xlo, int xhi, int ylo, int yhi) {
  if (!o) return ORC_EINVAL;
  int v[4] = {xlo, xhi, ylo, yhi};
  for (int k = 0; k < 4; ++k) {
    if (v[k] < 0 || v[k] > 2) return ORC_EINVAL;
    o->wall[k] = v[k];
  }
  return ORC_OK;
}

/* Boundary ghosts, 3 layers (reading #14): on a solid wall ghost -1-k mirrors cell k
 * (H, b, W copied, the normal momentum negated, the tangential copied); on an open
 * (zero-gradient, NEXT-4) side every ghost layer copies the boundary cell unchanged.
 * x-ghosts first on every padded row (owned rows and caller-supplied halo rows),
 * then y-ghosts over the full padded width (corners compose both rules). */
static void ghost_copy(orc_t* o, size_t d, size_t s, int negx, int negy) {
  o->H[d] = o->H[s]; o->b[d] = o->b[s]; o->W[d] = o->W[s];
  o->Qx[d] = negx ? -o->Qx[s] : o->Qx[s];
  o->Qy[d] = negy ? -o->Qy[s] : o->Qy[s];
}

static void mirror_fill(orc_t* o) {
  int nx = o->nx, ny = o->ny;
  for (int j = -G; j < ny + G; ++j) {
    for (int k = 0; k < G; ++k) {
      if (o->wall[0] == 1) ghost_copy(o, IDX(o, -1 - k, j), IDX(o, k, j), 1, 0);
      if (o->wall[0] == 2) ghost_copy(o, IDX(o, -1 - k, j), IDX(o, 0, j), 0, 0);
      if (o->wall[1] == 1) ghost_copy(o, IDX(o, nx + k, j), IDX(o, nx - 1 - k, j), 1, 0);
      if (o->wall[1] == 2) ghost_copy(o, IDX(o, nx + k, j), IDX(o, nx - 1, j), 0, 0);
    }
  }
  for (int i = -G; i < nx + G; ++i) {
    for (int k = 0; k < G; ++k) {
      if (o->wall[2] == 1) ghost_copy(o, IDX(o, i, -1 - k), IDX(o, i, k), 0, 1);
      if (o->wall[2] == 2) ghost_copy(o, IDX(o, i, -1 - k), IDX(o, i, 0), 0, 0);
      if (o->wall[3] == 1) ghost_copy(o, IDX(o, i, ny + k), IDX(o, i, ny - 1 - k), 0, 1);
      if (o->wall[3] == 2) ghost_copy(o, IDX(o, i, ny + k), IDX(o, i, ny - 1), 0, 0);
    }
  }
}

/* A_J of cell c at depth H: the constant, or Eq.4 with the cell's n_M (NEXT-4) */
static real cell_aj(const orc_t* o, size_t c, real H) {
  if (o->p.aj_mode == 0) return o->A_J;
  if (!(H > o->eps)) return RL(0);
  real n = o->fields_fric ? o->nfld[c] : RL(o->p.n_manning);
  return r_aj_eq4(o->g, n, o->s_rel, H, o->d50);
}

/* Step 9: maxima over the owned wet cells of the state, computed in the
 * working precision and widened exactly to double. */
static void reduce_M(orc_t* o, const real* H, const real* Qx, const real* Qy, double M[3]) {
  const orc_params* p = &o->p;
  real M1 = RL(0), M2 = RL(0), M3 = RL(0);
  for (int j = 0; j < o->ny; ++j) {
    for (int i = 0; i < o->nx; ++i) {
      size_t c = IDX(o, i, j);
      real Hc = H[c];
      if (!(Hc > o->eps)) continue;
      real r = RL(1) / Hc;
      real u = Qx[c] * r, v = Qy[c] * r;
      real s2 = u * u + v * v;
      real a = SQRT(s2);
      real t1 = s2;
      real t2 = a + SQRT(o->g * Hc);
      real t3 = RL(0);
      if (r_shamov_gate(o->kappa, s2, Hc, o->C_Sh) && r_bed_mobile(Hc, o->hbm)) {
        real pw = grass_pow(p->m_grass, p->m_real, s2, a);  /* |v|^m; m = 2: pw = s2 */
        t3 = ((cell_aj(o, c, Hc) * pw) * a) * o->W[c];
      }
      /* max that lets NaN win */
      if (!(t1 <= M1)) M1 = t1;
      if (!(t2 <= M2)) M2 = t2;
      if (!(t3 <= M3)) M3 = t3;
    }
  }
  M[0] = M1; M[1] = M2; M[2] = M3;
}

static int finite_all(const double* a, size_t n) {
  for (size_t k = 0; k < n; ++k)
    if (!isfinite(a[k])) return 0;
  return 1;
}

int orc_set_state(orc_t* o, const double* h, const double* hu, const double* hv,
                  const double* b, const double* psi) {
  if (!o || !h || !hu || !hv || !b) return ORC_EINVAL;
  size_t n = (size_t)o->nx * o->ny;
  if (!finite_all(h, n) || !finite_all(hu, n) || !finite_all(hv, n) || !finite_all(b, n))
    return ORC_EINVAL;
  for (size_t k = 0; k < n; ++k) {
    if (h[k] < 0.0) return ORC_EINVAL;
    if (psi && !(psi[k] >= 0.0 && psi[k] < 1.0)) return ORC_EINVAL;
  }
  for (int j = 0; j < o->ny; ++j)
    for (int i = 0; i < o->nx; ++i) {
      size_t s = (size_t)j * o->nx + i, d = IDX(o, i, j);
      o->H[d] = RL(h[s]); o->Qx[d] = RL(hu[s]); o->Qy[d] = RL(hv[s]); o->b[d] = RL(b[s]);
      o->W[d] = RL(1.0 / (1.0 - (psi ? psi[s] : 0.0))); /* Eq.1: W = 1/(1-psi) */
    }
  mirror_fill(o);
  reduce_M(o, o->H, o->Qx, o->Qy, o->M);
  o->have_state = 1;
  o->t = 0.0; o->steps = 0; o->last_dt = 0.0;
  return ORC_OK;
}

int orc_set_state_padded(orc_t* o, const double* H, const double* Qx, const double* Qy,
                         const double* b, const double* W) {
  if (!o || !H || !Qx || !Qy || !b || !W) return ORC_EINVAL;
  size_t n = (size_t)o->pw * o->ph;
  for (size_t k = 0; k < n; ++k) {
    o->H[k] = RL(H[k]); o->Qx[k] = RL(Qx[k]); o->Qy[k] = RL(Qy[k]);
    o->b[k] = RL(b[k]); o->W[k] = RL(W[k]);
  }
  mirror_fill(o);
  reduce_M(o, o->H, o->Qx, o->Qy, o->M);
  o->have_state = 1;
  return ORC_OK;
}

/* NEXT-3: per-cell Manning n_M, absorption beta and
 * water source s >= 0 of Eq.6's sigma (rain, point inflow).  NULL
 * arrays mean: scalar n_M of the params, beta = 0, s = 0.  Arrays are [ny][nx]. */
int orc_set_fields(orc_t* o, const double* n_manning, const double* beta, const double* src) {
  if (!o) return ORC_EINVAL;
  size_t n = (size_t)o->nx * o->ny;
  for (size_t k = 0; k < n; ++k) {
    if (n_manning && !(n_manning[k] >= 0.0 && isfinite(n_manning[k]))) return ORC_EINVAL;
    if (beta && !(beta[k] >= 0.0 && isfinite(beta[k]))) return ORC_EINVAL;
    if (src && !(src[k] >= 0.0 && isfinite(src[k]))) return ORC_EINVAL;
  }
  for (int j = 0; j < o->ny; ++j)
    for (int i = 0; i < o->nx; ++i) {
      size_t s = (size_t)j * o->nx + i, d = IDX(o, i, j);
      double nm = n_manning ? n_manning[s] : o->p.n_manning;
      o->cg[d] = RL(o->p.g * (nm * nm));
      o->nfld[d] = RL(nm);
      o->beta[d] = RL(beta ? beta[s] : 0.0);
      o->srcf[d] = RL(src ? src[s] : 0.0);
    }
  /* the fields are mirrored into the wall ghosts like H and b (reading #14) */
  {
    real* fl[4] = {o->cg, o->beta, o->srcf, o->nfld};
    for (int q = 0; q < 4; ++q) {
      real* f = fl[q];
      for (int j = 0; j < o->ny; ++j)
        for (int k = 0; k < G; ++k) {
          if (o->wall[0]) f[IDX(o, -1 - k, j)] = f[IDX(o, o->wall[0] == 2 ? 0 : k, j)];
          if (o->wall[1])
            f[IDX(o, o->nx + k, j)] = f[IDX(o, o->wall[1] == 2 ? o->nx - 1 : o->nx - 1 - k, j)];
        }
      for (int i = -G; i < o->nx + G; ++i)
        for (int k = 0; k < G; ++k) {
          if (o->wall[2]) f[IDX(o, i, -1 - k)] = f[IDX(o, i, o->wall[2] == 2 ? 0 : k)];
          if (o->wall[3])
            f[IDX(o, i, o->ny + k)] = f[IDX(o, i, o->wall[3] == 2 ? o->ny - 1 : o->ny - 1 - k)];
        }
    }
  }
  o->has_fields = (n_manning || beta || src) ? 1 : 0;
  o->fields_fric = n_manning != NULL;
  o->fields_src = (beta || src) ? 1 : 0;
  return ORC_OK;
}

int orc_get_state(orc_t* o, double* h, double* hu, double* hv, double* b) {
  if (!o) return ORC_EINVAL;
  if (!o->have_state) return ORC_ENOSTATE;
  for (int j = 0; j < o->ny; ++j)
    for (int i = 0; i < o->nx; ++i) {
      size_t d = (size_t)j * o->nx + i, s = IDX(o, i, j);
      if (h) h[d] = o->H[s];
      if (hu) hu[d] = o->Qx[s];
      if (hv) hv[d] = o->Qy[s];
      if (b) b[d] = o->b[s];
    }
  return ORC_OK;
}

int orc_get_state_padded(orc_t* o, double* H, double* Qx, double* Qy, double* b) {
  if (!o) return ORC_EINVAL;
  if (!o->have_state) return ORC_ENOSTATE;
  size_t n = (size_t)o->pw * o->ph;
  for (size_t k = 0; k < n; ++k) {
    if (H) H[k] = o->H[k];
    if (Qx) Qx[k] = o->Qx[k];
    if (Qy) Qy[k] = o->Qy[k];
    if (b) b[k] = o->b[k];
  }
  return ORC_OK;
}

int orc_reduce_M(orc_t* o, double M[3]) {
  if (!o) return ORC_EINVAL;
  if (!o->have_state) return ORC_ENOSTATE;
  reduce_M(o, o->H, o->Qx, o->Qy, M);
  return ORC_OK;
}

/* Step 0 -- K3, Eq.7, reading #9 */
int orc_tau_from_M(const orc_t* o, const double M[3], double* tau, int* lim) {
  if (!isfinite(M[0]) || !isfinite(M[1]) || !isfinite(M[2])) return ORC_ENONFINITE;
  double h = o->h;
  double t1 = h / (2.0 * sqrt(M[0]));
  double t2 = h / M[1];
  double t3 = (h * h) / (2.0 * M[2]);
  double m = t1;
  int l = 0;
  if (t2 < m) { m = t2; l = 1; }
  if (t3 < m) { m = t3; l = 2; }
  double T = o->p.K * m;
  if (o->p.dt_max < T) { T = o->p.dt_max; l = 3; }
  if (!isfinite(T)) return ORC_EDRY;
  *tau = T;
  if (lim) *lim = l;
  return ORC_OK;
}

/* ---- one step of R with a given tau ---------------------------------------- */

int orc_step_tau(orc_t* o, double tau_d) {
  if (!o) return ORC_EINVAL;
  if (!o->have_state) return ORC_ENOSTATE;
  const orc_params* p = &o->p;
  const int nx = o->nx, ny = o->ny;
  const real eps = o->eps;
  /* tau in the working precision; lambda = tau/h formed in double, then rounded once */
  const real tau = RL(tau_d);
  const real theta = RL(0.5) * tau;
  const real lam = RL(tau_d / o->h);
  const int fric = p->n_manning > 0.0 || o->fields_fric;
  real *H = o->H, *Qx = o->Qx, *Qy = o->Qy, *b = o->b, *W = o->W;
  const size_t sx = 1, sy = (size_t)o->pw;

  /* Step 1 -- K1: wet mask, eta, velocities on every cell */
  for (int j = -G; j < ny + G; ++j)
    for (int i = -G; i < nx + G; ++i) {
      size_t c = IDX(o, i, j);
      o->w[c] = H[c] > eps;
      o->eta[c] = H[c] + b[c];
      if (o->w[c]) {
        o->r[c] = RL(1) / H[c];
        o->u[c] = Qx[c] * o->r[c];
        o->v[c] = Qy[c] * o->r[c];
      } else {
        o->r[c] = RL(0); o->u[c] = RL(0); o->v[c] = RL(0);
      }
    }

  /* Step 2 -- K2: forces at t_n and friction gamma */
  for (int j = -G + 1; j < ny + G - 1; ++j)
    for (int i = -G + 1; i < nx + G - 1; ++i) {
      size_t c = IDX(o, i, j);
      if (!o->w[c]) { o->phix[c] = RL(0); o->phiy[c] = RL(0); o->gam[c] = RL(0); continue; }
      size_t e = c + sx, wv = c - sx, nn = c + sy, s = c - sy;
      real PE = face_force(o->cPh, o->eta[c], b[c], o->eta[e], b[e]);
      real PW = face_force(o->cPh, o->eta[wv], b[wv], o->eta[c], b[c]);
      real PN = face_force(o->cPh, o->eta[c], b[c], o->eta[nn], b[nn]);
      real PS = face_force(o->cPh, o->eta[s], b[s], o->eta[c], b[c]);
      o->phix[c] = -(PE + PW);
      o->phiy[c] = -(PN + PS);
      if (o->fields_fric) {
        /* friction field: c_gam = g n_M(x,y)^2 per cell (gamma = 0 where n_M = 0) */
        real sp = SQRT(o->u[c] * o->u[c] + o->v[c] * o->v[c]);
        o->gam[c] = (o->cg[c] * sp) * (o->r[c] * r_icbrt(H[c]));
      } else if (fric) {
        real sp = SQRT(o->u[c] * o->u[c] + o->v[c] * o->v[c]);
        o->gam[c] = (o->cgam * sp) * (o->r[c] * r_icbrt(H[c]));
      } else {
        o->gam[c] = RL(0);
      }
    }

  /* Step 3 -- K4: predictor to t_{n+1/2} */
  for (int j = -G + 1; j < ny + G - 1; ++j)
    for (int i = -G + 1; i < nx + G - 1; ++i) {
      size_t c = IDX(o, i, j);
      if (!o->w[c]) { o->Hh[c] = H[c]; o->ut[c] = RL(0); o->vt[c] = RL(0); continue; }
      real div = ((o->u[c + sx] - o->u[c - sx]) + (o->v[c + sy] - o->v[c - sy])) * o->inv_2h;
      o->Hh[c] = H[c] * FMA(-theta, div, RL(1));
      real f = RL(1) / FMA(theta, o->gam[c], RL(1));
      o->ut[c] = (FMA(theta, o->phix[c], Qx[c]) * f) * o->r[c];
      o->vt[c] = (FMA(theta, o->phiy[c], Qy[c]) * f) * o->r[c];
    }

  /* Step 4 -- K5: forces at t_{n+1/2} from eta_half, step-n mask */
  for (int j = -G + 2; j < ny + G - 2; ++j)
    for (int i = -G + 2; i < nx + G - 2; ++i) {
      size_t c = IDX(o, i, j);
      if (!o->w[c]) { o->phix2[c] = RL(0); o->phiy2[c] = RL(0); continue; }
      size_t e = c + sx, wv = c - sx, nn = c + sy, s = c - sy;
      real ec = o->Hh[c] + b[c];
      real PE = face_force(o->cPh, ec, b[c], o->Hh[e] + b[e], b[e]);
      real PW = face_force(o->cPh, o->Hh[wv] + b[wv], b[wv], ec, b[c]);
      real PN = face_force(o->cPh, ec, b[c], o->Hh[nn] + b[nn], b[nn]);
      real PS = face_force(o->cPh, o->Hh[s] + b[s], b[s], ec, b[c]);
      o->phix2[c] = -(PE + PW);
      o->phiy2[c] = -(PN + PS);
    }

  /* Step 5 -- K6: corrector momenta Q^L */
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      size_t c = IDX(o, i, j);
      if (!o->w[c]) { o->QLx[c] = RL(0); o->QLy[c] = RL(0); continue; }
      real f = RL(1) / FMA(tau, o->gam[c], RL(1));
      o->QLx[c] = FMA(tau, o->phix2[c], Qx[c]) * f;
      o->QLy[c] = FMA(tau, o->phiy2[c], Qy[c]) * f;
    }

  /* Step 7a: per-cell Grass flux J0 (Eq.3) gated by Shamov (Eq.5) from
   * (u~, v~, H) */
  for (int j = -G + 1; j < ny + G - 1; ++j)
    for (int i = -G + 1; i < nx + G - 1; ++i) {
      size_t c = IDX(o, i, j);
      real jx, jy, ja;
      r_grass_mr(cell_aj(o, c, H[c]), p->m_grass, p->m_real, o->ut[c], o->vt[c], &jx, &jy, &ja);
      real s2 = o->ut[c] * o->ut[c] + o->vt[c] * o->vt[c];
      if (r_shamov_gate(o->kappa, s2, H[c], o->C_Sh) && r_bed_mobile(H[c], o->hbm)) {
        o->J0x[c] = jx; o->J0y[c] = jy; o->J0a[c] = ja;
      } else {
        o->J0x[c] = RL(0); o->J0y[c] = RL(0); o->J0a[c] = RL(0);
      }
    }

  /* Steps 6-7 -- K7: minmod reconstruction of
   * (eta, H, u_n, u_t), hydrostatic step, HLL, sediment face flux.
   * x-faces: FH[(j, i)] is the face between cells (i-1, j) and (i, j). */
  for (int axis = 0; axis < 2; ++axis) {
    const size_t st = axis == 0 ? sx : sy;
    const real* un = axis == 0 ? o->ut : o->vt;
    const real* utn = axis == 0 ? o->vt : o->ut;
    const real* J0n = axis == 0 ? o->J0x : o->J0y;
    real* FH = axis == 0 ? o->FH : o->GH;
    real* FQn = axis == 0 ? o->FQx : o->GQy;
    real* FQt = axis == 0 ? o->FQy : o->GQx;
    real* FJ = axis == 0 ? o->FJ : o->GJ;
    int i_end = axis == 0 ? nx + 1 : nx;
    int j_end = axis == 0 ? ny : ny + 1;
    for (int j = 0; j < j_end; ++j)
      for (int i = 0; i < i_end; ++i) {
        size_t R = IDX(o, i, j), L = R - st;
        size_t LL = L - st, RR = R + st;
        real sL[4], sR[4];
        const real* q[4] = {o->eta, H, un, utn};
        for (int k = 0; k < 4; ++k) {
          sL[k] = r_minmod(q[k][L] - q[k][LL], q[k][R] - q[k][L]);
          sR[k] = r_minmod(q[k][R] - q[k][L], q[k][RR] - q[k][R]);
        }
        real qm[4], qp[4];
        /* face states q- = q_L + sigma_L/2, q+ = q_R - sigma_R/2 with one rounding each
         * (fma: exact product; = q + 0.5*sigma unless 0.5*sigma is subnormal) */
        for (int k = 0; k < 4; ++k) {
          qm[k] = FMA(RL(0.5), sL[k], q[k][L]);
          qp[k] = FMA(RL(-0.5), sR[k], q[k][R]);
        }
        real F[3];
        r_hll_face(o->g, qm[0], qm[1], qm[2], qm[3], qp[0], qp[1], qp[2], qp[3],
                   o->w[L], o->w[R], F);
        FH[R] = F[0]; FQn[R] = F[1]; FQt[R] = F[2];
        /* sediment face flux: donor by sign of u~_n,L + u~_n,R; tie averages */
        real Jn, Ja;
        if (!o->w[L] && !o->w[R]) {
          FJ[R] = RL(0);
          continue;
        }
        real us = un[L] + un[R];
        if (us > RL(0)) { Jn = J0n[L]; Ja = o->J0a[L]; }
        else if (us < RL(0)) { Jn = J0n[R]; Ja = o->J0a[R]; }
        else { Jn = RL(0.5) * (J0n[L] + J0n[R]); Ja = RL(0.5) * (o->J0a[L] + o->J0a[R]); }
        FJ[R] = r_slope_flux(Jn, Ja, o->C_J, (b[R] - b[L]) * o->inv_h);
      }
  }

  /* Step 8 -- K8 (Eq.1, Eq.6): conservative update */
  int neg = 0;
  const real src = o->src;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      size_t c = IDX(o, i, j);
      size_t e = c + sx, n = c + sy;
      real dH = (o->FH[e] - o->FH[c]) + (o->GH[n] - o->GH[c]);
      real dQx = (o->FQx[e] - o->FQx[c]) + (o->GQx[n] - o->GQx[c]);
      real dQy = (o->FQy[e] - o->FQy[c]) + (o->GQy[n] - o->GQy[c]);
      real dJ = (o->FJ[e] - o->FJ[c]) + (o->GJ[n] - o->GJ[c]);
      real Hn = FMA(-lam, dH, H[c]);
      real Qxn = FMA(-lam, dQx, o->QLx[c]);
      real Qyn = FMA(-lam, dQy, o->QLy[c]);
      if (o->fields_src) {
        /* sigma = s - beta H (reading #21): source explicit, absorption implicit,
         * H' = ((H - lam dF) + tau s) / (1 + tau beta); momenta scaled alike */
        real a = RL(1) / (RL(1) + tau * o->beta[c]);
        Hn = (Hn + tau * o->srcf[c]) * a;
        Qxn = Qxn * a;
        Qyn = Qyn * a;
      }
      real bn = FMA(-(lam * W[c]), dJ, b[c]) + (tau * W[c]) * src;
      if (!(Hn > eps)) { Qxn = RL(0); Qyn = RL(0); }
      if (Hn < -o->neg_tol) neg = 1;
      o->Hn[c] = Hn; o->Qxn[c] = Qxn; o->Qyn[c] = Qyn; o->bn[c] = bn;
    }
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      size_t c = IDX(o, i, j);
      H[c] = o->Hn[c]; Qx[c] = o->Qxn[c]; Qy[c] = o->Qyn[c]; b[c] = o->bn[c];
    }
  mirror_fill(o);

  /* Step 9: maxima for the next step's Eq.7 */
  reduce_M(o, H, Qx, Qy, o->M);
  o->t += tau_d;
  o->last_dt = tau_d;
  o->steps += 1;
  return neg ? ORC_ENEGDEPTH : ORC_OK;
}

int orc_step(orc_t* o, int nsteps, double* dt_log, int* lim_log, int* n_done) {
  if (!o || nsteps < 0) return ORC_EINVAL;
  if (!o->have_state) return ORC_ENOSTATE;
  int k = 0, st = ORC_OK;
  for (; k < nsteps; ++k) {
    double tau;
    int lim;
    st = orc_tau_from_M(o, o->M, &tau, &lim);
    if (st != ORC_OK) break;
    if (dt_log) dt_log[k] = tau;
    if (lim_log) lim_log[k] = lim;
    st = orc_step_tau(o, tau);
    if (st != ORC_OK) { ++k; break; }
  }
  if (n_done) *n_done = k;
  return st;
}

int orc_get_time(const orc_t* o, double* t, long long* steps, double* last_dt) {
  if (!o) return ORC_EINVAL;
  if (t) *t = o->t;
  if (steps) *steps = o->steps;
  if (last_dt) *last_dt = o->last_dt;
  return ORC_OK;
}

int orc_get_debug(const orc_t* o, const char* name, double* out) {
  if (!o || !name || !out) return ORC_EINVAL;
  size_t n = (size_t)o->pw * o->ph;
  if (strcmp(name, "w") == 0) {
    for (size_t k = 0; k < n; ++k) out[k] = o->w[k];
    return ORC_OK;
  }
  struct { const char* nm; const real* a; } tab[] = {
      {"eta", o->eta}, {"u", o->u}, {"v", o->v}, {"phix", o->phix}, {"phiy", o->phiy},
      {"gam", o->gam}, {"Hh", o->Hh}, {"ut", o->ut}, {"vt", o->vt}, {"phix2", o->phix2},
      {"phiy2", o->phiy2}, {"QLx", o->QLx}, {"QLy", o->QLy}, {"J0x", o->J0x},
      {"J0y", o->J0y}, {"J0a", o->J0a}, {"FH", o->FH}, {"FQx", o->FQx}, {"FQy", o->FQy},
      {"FJ", o->FJ}, {"GH", o->GH}, {"GQx", o->GQx}, {"GQy", o->GQy}, {"GJ", o->GJ},
      {"W", o->W}};
  for (size_t k = 0; k < sizeof(tab) / sizeof(tab[0]); ++k)
    if (strcmp(name, tab[k].nm) == 0) {
      for (size_t q = 0; q < n; ++q) out[q] = tab[k].a[q];
      return ORC_OK;
    }
  return ORC_EINVAL;
}
