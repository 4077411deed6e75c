/*
 * csph_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU implementation of the CSPH-TVD step of
 * Khrapov & Khoperskov, Lobachevskii J. Math. 41(8) 2020 (arXiv 2103.15196),
 * in the discrete reading "R" written out in DESIGN.md section 3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2103_15196_b200/) never links, imports or calls it, and shares no
 * code, header, constant or helper with it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (Eq. numbers in the
 * paper's order: Eq.1 Exner P:46-48, Eq.2 slope flux P:54-56, Eq.3 Grass
 * P:60-62, Eq.5 Shamov P:71-73, Eq.6 vector form P:76-108, Eq.7 timestep
 * P:114-119; kernels K1-K8 P:224-238).
 *
 * Parity-unpinned parts: the fidelity of R to the
 * authors' unpublished CSPH discretization (P:39, P:112 cite works that are
 * not in the reference), and Exner morphodynamics beyond the invariants.
 */
#ifndef CSPH_ORACLE_H
#define CSPH_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (same numeric meaning as the product ABI, defined here
 * independently). */
#define ORC_OK          0
#define ORC_EINVAL     -1
#define ORC_ENOSTATE   -2
#define ORC_ENOMEM     -3
#define ORC_ENEGDEPTH  -6
#define ORC_ENONFINITE -7
#define ORC_EDRY       -8

typedef struct {
  double g;        /* gravity */
  double K;        /* Courant number of Eq.7, 0<K<1 */
  double eps_dry;  /* wet iff H > eps_dry ("H[ind]>Eps") */
  double dt_max;   /* cap on tau (may be +inf) */
  double neg_tol;  /* H' < -neg_tol -> ORC_ENEGDEPTH */
  double n_manning;/* Manning n_M; 0 = no friction */
  double A_J;      /* Grass coefficient, Eq.3 */
  int    m_grass;  /* Grass exponent; R implements 2 */
  double C_J;      /* Eq.2 slope coefficient */
  double C_Sh;     /* Eq.5 Shamov constant; 0 = no gate */
  double d50;      /* Eq.5 median grain size */
  double q_plus, q_minus; /* Eq.1 sources (scalars) */
  int    aj_mode;  /* NEXT-4: 0 constant A_J; 1 Eq.4 A_J = 0.05 n_M^3/((s-1) sqrt(gH) d50) */
  double s_rel;    /* Eq.4 relative density rho_s/rho (> 1 in mode 1) */
  double h_bed_min;/* reading #31: no bedload where H <= h_bed_min; < 0 means d50 */
  double m_real;   /* NEXT-4: real Grass exponent in [0, 8] by the pinned pow; < 0: m_grass */
} orc_params;

typedef struct orc orc_t;

/* side index: 0 = x-low (i=-1..-3), 1 = x-high, 2 = y-low, 3 = y-high */
orc_t* orc_create(int nx, int ny, double dx, const orc_params* p);
void   orc_destroy(orc_t*);
/* per side: 1 = solid wall (3-layer mirror ghosts), 2 = open (zero-gradient ghosts,
 * NEXT-4), 0 = ghosts supplied by the caller */
int    orc_set_walls(orc_t*, int xlo, int xhi, int ylo, int yhi);
/* interior arrays [ny][nx]; psi may be NULL (psi = 0) */
int    orc_set_state(orc_t*, const double* h, const double* hu,
                     const double* hv, const double* b, const double* psi);
/* padded arrays [(ny+6)][(nx+6)] including the 3 ghost layers; W = 1/(1-psi) */
int    orc_set_state_padded(orc_t*, const double* H, const double* Qx,
                            const double* Qy, const double* b, const double* W);
int    orc_get_state(orc_t*, double* h, double* hu, double* hv, double* b);
/* NEXT-3: Manning field, absorption field, source field (each may be NULL) */
int    orc_set_fields(orc_t*, const double* n_manning, const double* beta, const double* src);
int    orc_get_state_padded(orc_t*, double* H, double* Qx, double* Qy, double* b);
/* maxima M1..M3 (step 9) of the current state over the owned cells */
int    orc_reduce_M(orc_t*, double M[3]);
/* step 0: tau from M; returns status; lim = argmin term (0..3) */
int    orc_tau_from_M(const orc_t*, const double M[3], double* tau, int* lim);
/* one step with an externally supplied tau (ghost refill only on wall sides) */
int    orc_step_tau(orc_t*, double tau);
/* nsteps full steps (tau from the state each step); logs may be NULL */
int    orc_step(orc_t*, int nsteps, double* dt_log, int* lim_log, int* n_done);
int    orc_get_time(const orc_t*, double* t, long long* steps, double* last_dt);

/* Intermediate arrays of the last step, padded layout (ny+6)x(nx+6).
 * names: "eta","u","v","w","phix","phiy","gam","Hh","ut","vt","phix2","phiy2",
 *        "QLx","QLy","J0x","J0y","J0a".
 * x-face arrays "FH","FQx","FQy","FJ": entry (j,i) = face between cells i-1 and i.
 * y-face arrays "GH","GQx","GQy","GJ": entry (j,i) = face between rows j-1 and j. */
int    orc_get_debug(const orc_t*, const char* name, double* out);

/* Closed-form pieces exposed for pins (same code the step uses). */
void   orc_grass(double A_J, double vx, double vy, double* jx, double* jy, double* jabs);
/* Eq.3 with an integer exponent m (0..8): |v|^m = s2^(m/2) [* sqrt(s2) if m odd] */
void   orc_grass_m(double A, int m, double vx, double vy, double* jx, double* jy, double* jabs);
/* Eq.4: A_J = (0.05 n^3) / (((s-1) sqrt(g H)) d50) */
double orc_aj_eq4(double g, double n_manning, double s_rel, double H, double d50);
double orc_slope_flux(double J0n, double J0abs, double C_J, double db_dn);
double orc_icbrt(double x);                   /* pinned x^(-1/3) recipe */
double orc_pow_pinned(double x, double q);    /* pinned x^q, x >= 0, q >= 0 */
double orc_gamma(const orc_params* p, double H, double u, double v); /* Manning gamma */
double orc_minmod(double a, double b);
/* Hydrostatic step + HLL on the advective flux of Eq.6 for one face, from the
 * reconstructed face states q- (left) and q+ (right); wL/wR = cell wet flags.
 * out[3] = (mass, normal momentum, tangential momentum) flux. */
void   orc_hll_face(double g, double eta_m, double H_m, double un_m, double ut_m,
                    double eta_p, double H_p, double un_p, double ut_p,
                    int wL, int wR, double out[3]);
int    orc_shamov_gate(double kappa, double s2, double H, double C_Sh);
/* reading #31: bedload only where H > h_bed_min (default d50) */
int    orc_bed_mobile(double H, double h_bed_min);

#ifdef __cplusplus
}
#endif
#endif
