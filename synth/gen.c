/*
 * synth/gen.c -- seeded synthetic inputs for the CSPH-TVD workloads.
 *
 * Shared by the tests, the oracle runs and the GPU runs.  It holds none of
 * the method's arithmetic: it only builds initial states (bed b, depth H,
 * momenta, porosity psi) shaped like the paper's workloads (DESIGN.md
 * section 6), from a counter-based hash, so the same bytes come out for the
 * same (config, size, window) on any x86-64 host with the same libm.
 *
 * hash(seed,i,j,o) = splitmix64(seed ^ i*0x9E3779B97F4A7C15
 *                               ^ j*0xC2B2AE3D27D4EB4F ^ o*0x165667B19E3779F9)
 * u = (hash >> 11) * 2^-53 in [0,1).
 * value noise: smoothstep-bilinear lattice of period P (cells);
 * fBm(P0, O) = sum_{o<O} 0.5^o (2 noise(P0/2^o) - 1).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

double syn_hash_u(uint64_t seed, int64_t i, int64_t j, int64_t o) {
  uint64_t k = seed ^ ((uint64_t)i * 0x9E3779B97F4A7C15ull) ^
               ((uint64_t)j * 0xC2B2AE3D27D4EB4Full) ^ ((uint64_t)o * 0x165667B19E3779F9ull);
  return (double)(splitmix64(k) >> 11) * (1.0 / 9007199254740992.0);
}

static double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

/* value noise in [0,1) at integer cell (i, j), lattice period P >= 1 */
double syn_noise(uint64_t seed, int64_t oct, int64_t P, int64_t i, int64_t j) {
  int64_t I = i >= 0 ? i / P : -((-i + P - 1) / P);
  int64_t J = j >= 0 ? j / P : -((-j + P - 1) / P);
  double fx = (double)(i - I * P) / (double)P;
  double fy = (double)(j - J * P) / (double)P;
  double sx = smooth(fx), sy = smooth(fy);
  double a = syn_hash_u(seed, I, J, oct), b = syn_hash_u(seed, I + 1, J, oct);
  double c = syn_hash_u(seed, I, J + 1, oct), d = syn_hash_u(seed, I + 1, J + 1, oct);
  double lo = (1.0 - sx) * a + sx * b;
  double hi = (1.0 - sx) * c + sx * d;
  return (1.0 - sy) * lo + sy * hi;
}

double syn_fbm(uint64_t seed, int64_t P0, int octaves, int64_t i, int64_t j) {
  double s = 0.0, amp = 1.0;
  int64_t P = P0;
  for (int o = 0; o < octaves; ++o) {
    if (P < 1) P = 1;
    s += amp * (2.0 * syn_noise(seed, o, P, i, j) - 1.0);
    amp *= 0.5;
    P /= 2;
  }
  return s;
}

/* fBm along one row j for i = 0..nx-1, identical values to syn_fbm(): the
 * lattice corner hashes are recomputed only when the lattice cell changes. */
static void fbm_row(uint64_t seed, int64_t P0, int octaves, int64_t j, int64_t nx,
                    double* out) {
  for (int64_t i = 0; i < nx; ++i) out[i] = 0.0;
  double amp = 1.0;
  int64_t P = P0;
  for (int o = 0; o < octaves; ++o) {
    if (P < 1) P = 1;
    int64_t J = j >= 0 ? j / P : -((-j + P - 1) / P);
    double fy = (double)(j - J * P) / (double)P;
    double sy = smooth(fy);
    int64_t Ic = -1;
    double a = 0, b = 0, c = 0, d = 0;
    for (int64_t i = 0; i < nx; ++i) {
      int64_t I = i / P;
      if (I != Ic) {
        Ic = I;
        a = syn_hash_u(seed, I, J, o); b = syn_hash_u(seed, I + 1, J, o);
        c = syn_hash_u(seed, I, J + 1, o); d = syn_hash_u(seed, I + 1, J + 1, o);
      }
      double fx = (double)(i - I * P) / (double)P;
      double sx = smooth(fx);
      double lo = (1.0 - sx) * a + sx * b;
      double hi = (1.0 - sx) * c + sx * d;
      double nz = (1.0 - sy) * lo + sy * hi;
      out[i] += amp * (2.0 * nz - 1.0);
    }
    amp *= 0.5;
    P /= 2;
  }
}

static double q20(double x) { return nearbyint(x * 1048576.0) / 1048576.0; }

static int64_t scl(int64_t v, int64_t n, int64_t ref) { return (v * n + ref / 2) / ref; }

/*
 * Fill rows [j0, j1) (global row index) of config `cfg` at global size nx x ny.
 * Output arrays are [(j1-j0)][nx].  Returns 0, or -1 for an unknown config.
 *   cfg 1: C1 dam break 1D-like (flat bed, H=1 | 0), variant 1 = Stoker (1 | 0.1)
 *   cfg 2: C2 lake at rest over rough terrain (variant 0 dyadic, 1 non-dyadic)
 *   cfg 3: C3 dam break over an erodible bed, dam with a breach
 *   cfg 4: C4 valley with dam across rows and a channel; variant 1 = C4D, the dam breached
 *   cfg 5: C5 river-floodplain flood, heterogeneous psi
 * Features are laid out on the reference sizes (C2 1024, C3 4096, C4 8192,
 * C5 16384) and scaled proportionally to the requested nx, ny.
 */
int syn_fill(int cfg, int variant, int64_t nx, int64_t ny, int64_t j0, int64_t j1,
             double* h, double* hu, double* hv, double* b, double* psi) {
  const double two_pi = 6.283185307179586;
  if (cfg < 1 || cfg > 5) return -1;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = j0; j < j1; ++j) {
    /* per-row fBm scratch lives in the output psi/hu rows until overwritten */
    double* F = hu + (size_t)(j - j0) * (size_t)nx; /* fBm of this row */
    double* N = hv + (size_t)(j - j0) * (size_t)nx; /* value noise of this row */
    if (cfg == 2) fbm_row(2, (int64_t)(256.0 * ((double)nx / 1024.0) + 0.5), 4, j, nx, F);
    else if (cfg == 3) fbm_row(4, scl(512, nx, 4096), 4, j, nx, F);
    else if (cfg == 4) fbm_row(5, scl(1024, nx, 8192), 4, j, nx, F);
    else if (cfg == 5) {
      fbm_row(6, scl(2048, nx, 16384), 5, j, nx, F);
      int64_t P7 = scl(512, nx, 16384) > 0 ? scl(512, nx, 16384) : 1;
      fbm_row(7, P7, 1, j, nx, N); /* 2*noise-1 */
    }
    for (int64_t i = 0; i < nx; ++i) {
      size_t k = (size_t)(j - j0) * (size_t)nx + (size_t)i;
      double H = 0.0, B = 0.0, PS = 0.4, QX = 0.0, QY = 0.0;
      if (cfg == 1) {
        B = 0.0;
        H = (i < nx / 2) ? 1.0 : (variant == 1 ? 0.1 : 0.0);
      } else if (cfg == 2) {
        double s = (double)nx / 1024.0;
        int64_t P = (int64_t)(256.0 * s + 0.5);
        (void)P;
        double bb = 1.0 + 1.2 * F[i] +
                    0.05 * (2.0 * syn_hash_u(3, i, j, 0) - 1.0);
        double eta0 = 1.3;
        if (variant == 0) { bb = q20(bb); eta0 = q20(eta0); }
        B = bb;
        H = eta0 - B;
        if (H < 0.0) H = 0.0;
      } else if (cfg == 3) {
        int64_t P = scl(512, nx, 4096);
        B = 0.0005 * (double)(scl(4096, nx, 4096) - i) * (4096.0 / (double)nx) +
            0.3 * F[i];
        (void)P;
        int64_t d0 = scl(1016, nx, 4096), d1 = scl(1024, nx, 4096);
        if (d1 <= d0) d1 = d0 + 1;
        int64_t r0 = scl(1792, ny, 4096), r1 = scl(2304, ny, 4096);
        int dam = (i >= d0 && i < d1) && !(j >= r0 && j < r1);
        if (dam) B = 10.0;
        if (i < d0) { H = 4.0 - B; if (H < 0.0) H = 0.0; }
      } else if (cfg == 4) {
        double s = (double)nx / 8192.0, sy = (double)ny / 8192.0;
        double jj = (double)j / sy; /* reference row coordinate */
        double xc = (4096.0 + 300.0 * sin(two_pi * jj / 4096.0)) * s;
        double dx = ((double)i - xc) / (4096.0 * s);
        int inch = fabs((double)i - xc) < 48.0 * s;
        B = 0.0005 * (8192.0 - jj) + 2.0 * dx * dx - (inch ? 2.0 : 0.0) +
            0.2 * F[i];
        int64_t d0 = scl(1016, ny, 8192), d1 = scl(1024, ny, 8192);
        if (d1 <= d0) d1 = d0 + 1;
        /* variant 1 (C4D): the dam has failed over a 1536 m breach around the channel at
         * t = 0 -- the reservoir floods the valley floor downstream (moving fronts) */
        const int breach = variant == 1 && fabs((double)i - xc) < 768.0 * s;
        if (j >= d0 && j < d1 && !inch && !breach) B = 12.0;
        if (j < d0) { H = 6.5 - B; if (H < 0.0) H = 0.0; }
        else if (inch) H = 1.0;
      } else {
        double s = (double)nx / 16384.0, sy = (double)ny / 16384.0;
        double jj = (double)j / sy;
        double xc = (8192.0 + 1500.0 * sin(two_pi * jj / 8192.0) +
                     400.0 * sin(two_pi * jj / 2048.0 + 1.0)) * s;
        double trend = 0.0002 * (16384.0 - jj);
        double plain = trend + 3.0 * F[i];
        double dist = fabs((double)i - xc);
        double half = 48.0 * s;
        B = plain;
        if (dist < half) B = trend - 5.0;
        double eta = trend - 0.8; /* overbank flood, ~30 % of the plain wet */
        H = eta - B;
        if (H < 0.0) H = 0.0;
        PS = 0.35 + 0.1 * (0.5 * (N[i] + 1.0));
        /* river inflow: the channel carries a 1 m/s downstream current */
        if (dist < half) { QY = H * 1.0; }
      }
      h[k] = H; b[k] = B; hu[k] = QX; hv[k] = QY;
      if (psi) psi[k] = PS;
    }
  }
  return 0;
}
