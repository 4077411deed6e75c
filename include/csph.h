/*
 * csph.h -- C-ABI of the B200-native CSPH-TVD step (arXiv 2103.15196).
 *
 * The library computes the per-timestep CSPH-TVD update of the coupled
 * Saint-Venant + Exner system (Eq.6, with the Exner
 * equation Eq.1) on a 2D structured grid, in the discrete
 * reading R of DESIGN.md section 3, entirely in CUDA kernels for sm_100a:
 *   K1 wet mask, K2 forces at t_n (:226), K3 timestep
 *   Eq.7 (:114-119, :228), K4 predictor (:230), K5 forces at t_{n+1/2} (:232),
 *   K6 corrector (:234), K7 face fluxes: minmod reconstruction + HLL in x and
 *   y (:236, :261-263) with the bedload flux Eqs.2,3,5 (:54-73), K8 update
 *   (:238).
 *
 * Conventions
 *  - Host arrays are fp64, row-major [ny][nx] (x fastest, index j*nx + i),
 *    owned by the caller, read or written only during the call (synchronous
 *    copies).  The handle owns all device memory, streams, graphs and NCCL
 *    communicators; csph_destroy frees them.  A handle is not thread-safe.
 *  - State U = (H, Hu, Hv, b) of Eq.6: h = water depth [m],
 *    hu, hv = momenta [m^2/s], b = bed elevation [m]; psi = bed porosity of
 *    Eq.1 (0 <= psi < 1), may be NULL (psi = 0).
 *  - Boundaries: solid reflective walls on the four global edges (DESIGN.md
 *    reading #14), or open zero-gradient edges (params.open_bc).
 *  - Every function returns 0 (CSPH_OK) or a negative CSPH_E* code; the
 *    thread-local csph_last_error() describes the last failure.
 *  - There is no CPU fallback: with no CUDA device every call that needs one
 *    fails with CSPH_ECUDA.
 */
#ifndef CSPH_H
#define CSPH_H

#ifdef __cplusplus
extern "C" {
#endif

#define CSPH_OK          0
#define CSPH_EINVAL     -1  /* bad argument, NaN/Inf or negative depth input, psi not in [0,1) */
#define CSPH_ENOSTATE   -2  /* step/get before set_state */
#define CSPH_ENOMEM     -3  /* device allocation failed */
#define CSPH_ECUDA      -4  /* CUDA runtime error (message in csph_last_error) */
#define CSPH_ENCCL      -5  /* NCCL error */
#define CSPH_ENEGDEPTH  -6  /* H' < -neg_tol after a step; the state after that step is kept */
#define CSPH_ENONFINITE -7  /* a maximum of Eq.7 is NaN or Inf */
#define CSPH_EDRY       -8  /* no wet cell and dt_max = +inf: Eq.7 gives no finite tau */

#define CSPH_PATH_FUSED  0  /* one y-marching kernel per step (default) */
#define CSPH_PATH_STAGED 1  /* the paper's kernel split K1..K8, intermediates in HBM */

typedef struct csph csph_t;

typedef struct {
  double g;          /* gravity [m/s^2], default 9.81 */
  double K;          /* Courant number of Eq.7, 0 < K < 1, default 0.25 (reading #13) */
  double eps_dry;    /* a cell is wet iff h > eps_dry ("H>Eps"), default 1e-6 m */
  double dt_max;     /* cap on tau, default +INF */
  double neg_tol;    /* h' < -neg_tol -> CSPH_ENEGDEPTH, default 1e-12 m */
  double n_manning;  /* Manning n_M [s m^-1/3]; 0 disables friction */
  double A_J;        /* Grass coefficient of Eq.3; 0 disables transport */
  int    m_grass;    /* Grass exponent m of Eq.3, integer 0..8 (2 for fine sand) */
  double C_J;        /* Eq.2 slope coefficient (1.5..2.3, up to 5) */
  double C_Sh;       /* Eq.5 Shamov constant; 0 disables the gate */
  double d50;        /* Eq.5 median grain size [m] (> 0 when C_Sh > 0); by default also the
                        depth at or below which no bedload moves (h_bed_min below) */
  double q_plus;     /* Eq.1 deposition source [m/s], default 0 */
  double q_minus;    /* Eq.1 erosion drain [m/s], default 0 */
  int    precision;  /* 64 (default, fp64: the hot path, bitwise = the oracle) or 32 (NEXT-2
                        fp32 state and arithmetic, fused path, walls, m = 2, constant A_J;
                        DESIGN.md 3.14) */
  int    device;     /* CUDA ordinal for csph_create (single-process use) */
  int    path;       /* CSPH_PATH_FUSED (default) or CSPH_PATH_STAGED */
  int    tile_rows;  /* fused path: rows marched per CTA (= HGS tile height); 0 = auto:
                        at every set_state the largest of 192/128/64/32/16 whose wet tiles fill
                        2.5 waves of 3 resident CTAs per SM.  A pure
                        performance parameter: results are bitwise identical for any value */
  int    hgs;        /* 1 (default): skip tiles whose neighbourhood is dry (the paper's
                        HGS; exact); 0: march every tile */
  int    aj_mode;    /* 0 (default): constant A_J; 1: Eq.4
                        A_J = 0.05 n_M^3 / ((s-1) sqrt(g H) d50), H the local depth */
  double s_rel;      /* Eq.4 relative density rho_s/rho (> 1), default 2.65 */
  int    open_bc;    /* NEXT-4 boundaries: bit mask of open (zero-gradient) edges,
                        1 x-low, 2 x-high, 4 y-low, 8 y-high; default 0 = solid walls */
  int    graphs;     /* 1 (default): a single-grid handle replays its steps in pairs from
                        CUDA graphs (bitwise identical); 0: plain launches */
  double h_bed_min;  /* reading #31: no bedload (Eq.3 J0, Eq.7's bed term)
                        where H <= h_bed_min; < 0 (default -1) means h_bed_min = d50 (a water
                        column no deeper than the grain); 0 is the literal Eq.5 (any wet cell
                        may carry bedload) */
  double m_real;     /* Grass exponent as a real number (Eq.3, "A_J, m are the
                        constant coefficients"); < 0 (default -1): use the integer m_grass;
                        >= 0: |v|^m by the pinned pow of DESIGN.md 3.12 (fp64 only) */
  int    halo_push;  /* fused path, several strips: 1 (default) the step kernel
                        writes each strip's first / last 3 rows and facing tile flags
                        straight into the neighbouring strip's ghost rows (peer memory: a
                        strip of the same process, or another rank's GPU mapped through CUDA
                        IPC, csph_ipc_*); 0, or no peer access: peer copies (MULTI) / NCCL
                        send-recv (DIST) after the edge tile rows.  Bitwise identical. */
} csph_params;

/* Fill *p with the defaults above. */
void        csph_default_params(csph_params* p);

/* One grid of nx x ny cells of size dx [m] on one GPU (p->device).
 * Returns NULL on error (nx or ny < 3, dx <= 0, bad params, no CUDA device,
 * allocation failure) -> csph_last_error(). */
csph_t*     csph_create(int nx, int ny, double dx, const csph_params* p);

/* Upload the full state (global arrays [ny][nx]); computes W = 1/(1-psi),
 * the wall ghosts and the Eq.7 maxima of the initial state.  Validates
 * inputs: CSPH_EINVAL on NaN/Inf, h < 0 or psi outside [0,1).  In a
 * distributed handle each rank copies its own strip plus halo rows. */
int         csph_set_state(csph_t*, const double* h, const double* hu, const double* hv,
                           const double* b, const double* psi);

/* As csph_set_state, but the arrays hold only global rows [j_begin, j_end)
 * ([j_end-j_begin][nx]); they must cover this handle's owned rows and the 3
 * halo rows on each strip side that has a neighbour.  Lets each rank of a
 * distributed run generate only its own strip. */
int         csph_set_state_rows(csph_t*, int j_begin, int j_end, const double* h,
                                const double* hu, const double* hv, const double* b,
                                const double* psi);

/* NEXT-3 spatial inputs of the paper's model (Manning n_M(x,y) and
 * absorption beta(x,y); Eq.6's sigma): per-cell Manning
 * coefficient [s m^-1/3] (replaces params.n_manning), absorption rate beta [1/s]
 * and water source s >= 0 [m/s] (rain, point inflow).  sigma = s - beta*H enters
 * K8 as H' = ((H - lam dF) + tau s)/(1 + tau beta), momenta scaled by the same
 * factor.  Global arrays [ny][nx]; any may be NULL (n_M from
 * params; beta = s = 0).  Persist across csph_set_state. */
int         csph_set_fields(csph_t*, const double* n_manning, const double* beta,
                            const double* src);
/* Row-window variant (global rows [j_begin, j_end), covering owned rows + halo). */
int         csph_set_fields_rows(csph_t*, int j_begin, int j_end, const double* n_manning,
                                 const double* beta, const double* src);

/* Advance exactly nsteps CSPH-TVD steps, each with its own Eq.7 tau computed
 * on the device.  No host synchronisation inside the call except one status
 * readback at its end.  A single-grid handle replays pairs of steps from CUDA
 * graphs (captured on first use, rebuilt after set_state / set_fields;
 * params.graphs = 0 disables them).  On CSPH_ENEGDEPTH/ENONFINITE/EDRY the steps up to the
 * failing one are done (see csph_get_time) and later calls return the same code. */
int         csph_step(csph_t*, int nsteps);

/* Download the state into global-layout arrays [ny][nx] (any may be NULL).
 * A distributed handle writes only its owned rows. */
int         csph_get_state(csph_t*, double* h, double* hu, double* hv, double* b);

/* Download global rows [j_begin, j_end) that this handle owns into
 * [j_end-j_begin][nx] arrays. */
int         csph_get_state_rows(csph_t*, int j_begin, int j_end, double* h, double* hu,
                                double* hv, double* b);

/* Asynchronous Save (the "Save" block: states are recorded every
 * 100-1000 iterations, and CUDA streams separate the CPU<->GPU copies from the
 * computation).  Snapshots the state as of the last completed step into a
 * device buffer (dense fp64 [4][owned rows][nx], allocated on first use:
 * 32 B per owned cell), then copies it to the caller's global-layout arrays
 * [ny][nx] (owned rows only; any may be NULL) on a separate stream, and returns
 * without waiting.  csph_step calls made afterwards run concurrently with that
 * copy and do not change what it delivers.  The host arrays are the caller's
 * and must stay valid and untouched until csph_save_wait; pinned (page-locked)
 * arrays are needed for the copy to overlap the steps.  A second csph_save_begin
 * before csph_save_wait is ordered after the first on the device.  Errors:
 * CSPH_EINVAL (NULL handle), CSPH_ENOSTATE, CSPH_ENOMEM, CSPH_ECUDA. */
int         csph_save_begin(csph_t*, double* h, double* hu, double* hv, double* b);

/* Block until every csph_save_begin issued on this handle has landed in host
 * memory.  CSPH_OK when none is pending. */
int         csph_save_wait(csph_t*);

/* Simulated time t = sum of tau, steps done, last tau. */
int         csph_get_time(csph_t*, double* t, long long* steps_done, double* last_dt);

/* Copy the last min(cap, steps done) entries of the device dt log (tau of
 * each step, in order) and the Eq.7 limiter of each (0: h/(2 v_p),
 * 1: h/v_s, 2: h^2/(2D), 3: dt_max); *n = entries copied. */
int         csph_get_dt_log(csph_t*, double* dt, int* limiter, int cap, int* n);

/* Eq.7 maxima (M1 = max |v|^2, M2 = max(|v| + sqrt(gH)), M3 = max |J0|/(1-psi))
 * of the current state (after the allreduce in a distributed handle). */
int         csph_get_maxima(csph_t*, double M[3]);

/* Use the caller's cudaStream_t (e.g. torch's current stream) for all work. */
int         csph_set_stream(csph_t*, void* cuda_stream);

/* Rows [j0, j1) owned by `rank` of `nranks` in the row-strip partition of ny
 * rows ("Ny_dev"): the first ny % nranks ranks get one extra row.
 * Host-only; CSPH_EINVAL if a strip would have fewer than 3 rows. */
int         csph_strip_rows(int ny, int nranks, int rank, int* j0, int* j1);

/* Load-balanced row partition (host-only).  w[0..ny) are non-negative per-row costs
 * (e.g. the wet cells of each row plus a small per-row constant: the fused kernel's time
 * is set by its wet tiles).  Writes bounds[0..nranks] with bounds[0] = 0,
 * bounds[nranks] = ny, every strip >= 3 rows, minimising the largest strip cost (bisection
 * on it; feasibility by a reachability sweep, O(nranks * ny) per probe).  All-zero weights
 * give the even split.  CSPH_EINVAL
 * on a NULL pointer, a negative/NaN weight, or ny < 3 * nranks. */
int         csph_balance_rows(int ny, int nranks, const double* w, int* bounds);

/* Per-row cost weights of the CURRENT state for csph_balance_rows: for every row j
 * this handle owns (all rows of a single grid or MULTI handle; a DIST rank's own strip),
 * w[j] = (wet cells of row j, H > eps_dry) + 0.03 nx -- the fused kernel's cost of a full row
 * vs a dry one.  w is a host array of ny doubles indexed by the global row; entries of rows the
 * handle does not own are left untouched (a DIST harness all-gathers them).  Syncs with the
 * device.  CSPH_EINVAL on NULL, CSPH_ENOSTATE before set_state. */
int         csph_row_weights(csph_t*, double* w);

/* Re-partition a DIST or MULTI handle into the strips [bounds[r], bounds[r+1]) between two
 * steps (collective: every rank calls it with the same bounds, e.g. from csph_balance_rows on
 * all-gathered csph_row_weights).  The current state, W = 1/(1-psi) and the NEXT-3 fields
 * migrate between strips (NCCL send/recv of full padded rows for DIST, a rank's rows to itself
 * by a device copy; peer copies for MULTI); the control block (time, step count, tau of the
 * next step, status), the dt log and the tile height rule carry over; HGS tile flags restart
 * with every tile active (the first step marches all tiles).  Results are bitwise those of an
 * unpartitioned run.  CSPH_EINVAL on a SINGLE handle or bad bounds (as csph_create_dist_rows),
 * CSPH_ENOSTATE before set_state, CSPH_ENOMEM / CSPH_ECUDA / CSPH_ENCCL on failure (the
 * handle is then unusable). */
int         csph_rebalance_rows(csph_t*, const int* bounds);

void        csph_destroy(csph_t*);
const char* csph_strerror(int code);
const char* csph_last_error(void);

/* ---- multi-GPU: one process per GPU, row strips, NCCL over NVLink ------- */
/* Rank 0 makes the NCCL unique id; the harness broadcasts it (e.g. through
 * torch.distributed) and every rank calls csph_create_dist with it.  Once csph_ipc_link has
 * mapped the other ranks' buffers (params.halo_push = 1, fused path) a step
 * moves no data through NCCL: the step kernel's first / last tile rows write their 3 rows
 * (4 fields) and HGS band flags straight into the neighbours' ghost rows over NVLink, and
 * each rank's ctrl kernel publishes its Eq.7 maxima (and the negative-depth flag) into every
 * rank's inbox and combines them (max).  Without the link: ncclSend/ncclRecv of the halo
 * rows to ranks r-1, r+1 (no wrap-around, reading #18) after the edge tile rows, overlapped
 * with the interior, and ncclAllReduce(max) of the maxima. */
int         csph_nccl_id_bytes(void);
int         csph_make_nccl_id(void* out);
csph_t*     csph_create_dist(int nx, int ny, double dx, const csph_params* p,
                             int rank, int nranks, int local_device, const void* nccl_id);
/* The same with a caller-chosen partition: rank r owns rows [bounds[r], bounds[r+1])
 * (bounds[0..nranks], identical on every rank; e.g. from csph_balance_rows).  NULL and
 * CSPH_EINVAL (csph_last_error) unless 0 = bounds[0] < ... < bounds[nranks] = ny with every
 * strip >= 3 rows. */
csph_t*     csph_create_dist_rows(int nx, int ny, double dx, const csph_params* p,
                                  int rank, int nranks, const int* bounds, int local_device,
                                  const void* nccl_id);

/* DIST peer memory.  csph_ipc_export writes csph_ipc_blob_bytes() bytes
 * describing this rank's state buffers, ghost tile-flag rows and combine inbox (CUDA IPC
 * handles, strip geometry) into out (host memory).  The harness all-gathers the blobs and
 * every rank calls csph_ipc_link with all of them (nblobs = nranks, rank order, one after the
 * other in `blobs`): the neighbours' buffers and every rank's inbox are mapped
 * (cudaIpcOpenMemHandle, peer access enabled lazily) and the following steps push halos from
 * inside the kernel and combine the maxima in the ctrl kernels (see above).  Collective in
 * effect: every rank must link before the next step.  CSPH_EINVAL for a non-DIST handle, a
 * wrong count or a blob that is not rank r's strip (geometry checked), CSPH_ECUDA if a handle
 * cannot be opened (e.g. no peer access; the handle then keeps NCCL).  csph_ipc_link(h, NULL,
 * 0) drops the links (back to NCCL): every rank must use the same transport, so a harness
 * whose link failed on some rank unlinks on all.  A 1-rank handle needs no link.
 * csph_rebalance_rows drops the links (new buffers): link again. */
int         csph_ipc_blob_bytes(void);
int         csph_ipc_export(csph_t*, void* out);
int         csph_ipc_link(csph_t*, const void* blobs, int nblobs);

/* Single-process row-strip decomposition: nstrips strips on the devices
 * listed in `devices` (strips may share a device), halos pushed by the step kernel into the
 * neighbouring strips' ghost rows (params.halo_push = 1 and peer access between the devices;
 * otherwise copied with cudaMemcpyPeerAsync after the edge tile rows) and the maxima combined
 * on the first device.  The same strip kernels and halo layout as csph_create_dist
 * (PAPER.md:198-218's one-host-thread-drives-all-GPUs arrangement). */
csph_t*     csph_create_multi(int nx, int ny, double dx, const csph_params* p,
                              int nstrips, const int* devices);
/* The same with caller-chosen strip rows bounds[0..nstrips] (as csph_create_dist_rows). */
csph_t*     csph_create_multi_rows(int nx, int ny, double dx, const csph_params* p,
                                   int nstrips, const int* devices, const int* bounds);

/* Kernel timing (bench): when enabled, csph_step records CUDA events on the
 * handle's stream around each step's main kernel(s) (the fused step kernel, or
 * K1..K8 of the staged path) and accumulates their device time. */
int         csph_profile(csph_t*, int enable);
/* Accumulated main-kernel device time [ms] and number of steps timed since
 * profiling was enabled. */
int         csph_get_profile(csph_t*, double* main_kernel_ms, long long* steps_timed);

/* HGS tile counters of the fused path since csph_set_state (or the last reset):
 * counts[0] tiles marched, counts[1] tiles updated by an identity copy (dry
 * neighbourhood), counts[2] tiles skipped (dry and already identical in both
 * state buffers).  A tile is the 120-column x TY-row chunk one CTA owns (TY =
 * params.tile_rows, or chosen from the state at set_state). */
int         csph_get_tile_stats(csph_t*, long long counts[3]);
int         csph_reset_tile_stats(csph_t*);

/* Self-test: the kernels' branch-free correctly rounded reciprocal and square
 * root against IEEE division and sqrt on n hashed inputs
 * (and the tiny-argument square root on scaled ones); *mismatches must be 0. */
int         csph_selftest_math(long long n, unsigned long long seed, long long* mismatches);

/* Number of kernel launches the last csph_step issued (for the bench). */
long long   csph_last_launch_count(csph_t*);

#ifdef __cplusplus
}
#endif
#endif /* CSPH_H */
