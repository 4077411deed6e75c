// csph_api.cu -- the C-ABI of include/csph.h: handle lifecycle, HBM layout,
// set/get state, the per-step control kernel (Eq.7 on the device), wall ghosts,
// and the row-strip decomposition over NCCL (one process per GPU) or over
// cudaMemcpyPeer (one process driving several strips).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <functional>
#include <vector>

#include "../../include/csph.h"
#include "csph_launch.h"
#include "csph_real.cuh"

using namespace ck;

// ---------------------------------------------------------------- errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(CSPH_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                           \
  } while (0)

// ---------------------------------------------------------------- NCCL (lazy)

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    fail(CSPH_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
    return false;
  }
#define SYM(field, name)                                                \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) {                                                  \
    fail(CSPH_ENCCL, "libnccl lacks %s", name);                         \
    return false;                                                       \
  }
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(AllReduce, "ncclAllReduce");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g_nccl.ok = true;
  return true;
}
}  // namespace

#define NK(call)                                                                    \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess)                                                          \
      return fail(CSPH_ENCCL, "%s: %s", #call, g_nccl.GetErrorString(r_));          \
  } while (0)

// ---------------------------------------------------------------- handle

namespace {

struct Strip {
  int dev = 0;
  int gj0 = 0;           // global row of the first owned row
  StripView v{};
  Scratch scr{};
  bool has_scr = false;
  Ctrl* ctrl = nullptr;              // device
  unsigned long long* gM = nullptr;  // device accumulator [4]
  double* Mlast = nullptr;           // device [4]
  double* dtlog = nullptr;           // device [LOGCAP]
  int* limlog = nullptr;             // device [LOGCAP]
  int* dflags = nullptr;             // device validation flags
  unsigned char* tflag = nullptr;    // HGS tile wet flags [2][ntiles]
  int ty = 128;                      // rows per CTA tile of the fused kernel (= HGS tile)
  bool auto_ty = false;              // ty chosen from the state at set_state
  size_t tflag_cap = 0;              // tiles the flag buffers hold (finest tiling)
  unsigned char* wetblk = nullptr;   // auto_ty: wet flags of 120 x 16 blocks [ny/16][ntx]
  unsigned char* gflag = nullptr;    // neighbours' facing tile-row flags [2 parity][2 side][ntx]
  int nsm = 148;
  unsigned char* tstate = nullptr;   // HGS identity-copy counters [ntiles]
  unsigned long long* hstats = nullptr;  // HGS tile counters: marched, copied, skipped
  // launch order, by the state parity a step reads: tcost[p] per tile, the
  // full-cost rows of the step that read buffer p; torder[p] the order of the step reading
  // p, sorted on the order stream `ost` from tcost[p] of two steps before while the step
  // in between runs (ev_ofork / ev_ojoin; osort_pending: a sort not yet joined by st)
  unsigned short* tcost = nullptr;   // [2][tflag_cap]
  int* torder = nullptr;             // [2][tflag_cap]
  cudaStream_t ost = nullptr;
  cudaEvent_t ev_ofork = nullptr, ev_ojoin = nullptr;
  bool osort_pending = false;
  // peer combine: this strip's inbox [2][nranks][kInboxW] and the device array
  // of every rank's inbox pointer (own device memory; nullptr until linked)
  unsigned long long* inbox = nullptr;
  unsigned long long** dpeers = nullptr;
  int ntx = 0, nty = 0;
  double* Wbuf = nullptr;            // device psi -> W field (when psi varies)
  float* Wbuf32 = nullptr;           // fp32 mode W field
  double* tmpd = nullptr;            // fp32 mode: fp64 staging for get_state
  // asynchronous Save (csph_save_begin): dense fp64 snapshot [4][ny][nx] of the owned rows,
  // copied to the host on its own stream `sst` while later steps run on `st`
  double* snap = nullptr;
  cudaStream_t sst = nullptr;
  cudaEvent_t ev_snap = nullptr, ev_saved = nullptr;
  bool save_issued = false;  // ev_saved recorded at least once
  double *cgbuf = nullptr, *betabuf = nullptr, *srcbuf = nullptr;  // NEXT-3 fields
  double* ajbuf = nullptr;  // NEXT-4: 0.05 n_M^3 field for Eq.4
  cudaStream_t st = nullptr;
  bool own_stream = true;
  cudaEvent_t ev = nullptr;
  cudaStream_t cst = nullptr;                        // NCCL stream (DIST)
  cudaEvent_t ev_edge = nullptr, ev_int = nullptr, ev_comm = nullptr;
  std::vector<void*> allocs;
};

enum Mode { SINGLE = 0, DIST = 1, MULTI = 2 };

}  // namespace

struct csph {
  int nx = 0, ny = 0;
  double dx = 1.0;
  csph_params p{};
  Phys P{};
  Mode mode = SINGLE;
  int rank = 0, nranks = 1;
  std::vector<int> bounds;  // DIST: the strip bounds of every rank [nranks + 1]
  ncclComm_t comm = nullptr;
  std::vector<Strip> s;
  bool have_state = false;
  int host_parity = 0;  // buffer the next step reads (as launched)
  long long launches = 0;
  unsigned long long* gather = nullptr;  // MULTI: [nstrips*4] on strip 0's device
  // halo push: every interior strip edge is linked (StripView nH.. ngflag), so
  // the split step launches each strip whole and moves no halo rows itself
  bool push = false;
  // the Eq.7 maxima combined by the ctrl kernels over peer memory (no gather / allreduce)
  bool p2p_combine = false;
  std::vector<void*> ipc_open;  // DIST: neighbour buffers opened through CUDA IPC
  bool profiling = false;
  std::vector<cudaEvent_t> evs;  // pairs around the main kernel of each step (strip 0)
  double prof_ms = 0.0;
  long long prof_steps = 0;
  // single-grid handles replay steps in pairs from CUDA graphs (one per starting buffer
  // parity: the HGS flag buffers alternate); rebuilt after anything a launch bakes in
  // (state upload, spatial fields) changes.  CSPH_NO_GRAPHS=1 turns them off.
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  long long graph_kernels = 0;  // kernel launches inside one pair graph
  cudaStream_t cap = nullptr;   // private capture stream (the handle's may be the legacy default)
  bool graphs = true;  // csph_params.graphs
};

static void graphs_reset(csph* H) {
  for (auto& g : H->gexec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

static void graphs_free(csph* H) {
  graphs_reset(H);
  if (H->cap) cudaStreamDestroy(H->cap);
  H->cap = nullptr;
}

// ---------------------------------------------------------------- kernels

namespace {

constexpr int kTyMin = 16;  // finest automatic tiling (rows)

// The combine of the Eq.7 maxima and the negative-depth flag over peer memory:
// every strip / rank owns an inbox [2 slots][nranks][kInboxW] u64 that every other one can
// store to (same process, peer access, or CUDA IPC); peers[r] = rank r's inbox.
constexpr int kInboxW = 8;  // m0, m1, m2, neg, sequence number, pad
struct PeerCombine {
  unsigned long long* const* peers;  // [nranks] device array of inbox pointers, or nullptr
  unsigned long long* inbox;         // this rank's inbox
  int nranks, rank;
};

// Publish this rank's 4 partial maxima of the step just done into slot (step & 1) of every
// rank's inbox -- the values, a system-scope fence, then the sequence number step + 1 -- and
// wait until every rank's entry of that slot carries it; gM becomes the max over the ranks.
// Two slots suffice: a rank can publish step n+2 only after every rank has published n+1,
// which each does after its own read of step n.  Exact (u64 max of the bit patterns) and
// independent of arrival order.  A peer silent for 10 s sets CSPH_ENCCL.
__device__ int peer_combine(const PeerCombine& pc, unsigned long long* gM, long long step) {
  const int slot = (int)(step & 1);
  const unsigned long long seq = (unsigned long long)step + 1ull;
  for (int r = 0; r < pc.nranks; ++r) {
    unsigned long long* d = pc.peers[r] + ((size_t)slot * pc.nranks + pc.rank) * kInboxW;
    for (int k = 0; k < 4; ++k) d[k] = gM[k];
  }
  __threadfence_system();
  for (int r = 0; r < pc.nranks; ++r) {
    volatile unsigned long long* d =
        pc.peers[r] + ((size_t)slot * pc.nranks + pc.rank) * kInboxW;
    d[4] = seq;
  }
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned long long m[4] = {0, 0, 0, 0};
  for (int r = 0; r < pc.nranks; ++r) {
    volatile unsigned long long* e = pc.inbox + ((size_t)slot * pc.nranks + r) * kInboxW;
    while (e[4] != seq) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) return CSPH_ENCCL;
      __nanosleep(100);
    }
    __threadfence_system();
    for (int k = 0; k < 4; ++k) m[k] = e[k] > m[k] ? e[k] : m[k];
  }
  for (int k = 0; k < 4; ++k) gM[k] = m[k];
  return 0;
}

__global__ void ctrl_kernel(Ctrl* C, unsigned long long* gM, double* Mlast, double* dtlog,
                            int* limlog, Phys P, int advance, PeerCombine pc = PeerCombine{}) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (advance && pc.peers && C->status == 0) {
    const int e = peer_combine(pc, gM, C->step);
    if (e) {
      C->status = e;
      return;
    }
  }
  if (advance) {
    if (C->status == 0) {
      C->parity ^= 1;
      C->step += 1;
      C->t += C->tau;
      if (gM[3]) C->status = CSPH_ENEGDEPTH;  // any strip / rank (combined in gM[3])
    }
  }
  double M[3];
  for (int k = 0; k < 3; ++k) {
    M[k] = __longlong_as_double((long long)gM[k]);
    Mlast[k] = M[k];
    gM[k] = 0ull;
  }
  gM[3] = 0ull;
  if (C->status) return;
  if (!isfinite(M[0]) || !isfinite(M[1]) || !isfinite(M[2])) {
    C->status = CSPH_ENONFINITE;
    return;
  }
  // Step 0 -- K3, Eq.7
  double h = P.h;
  double t1 = h / (2.0 * sqrt(M[0]));
  double t2 = h / M[1];
  double t3 = (h * h) / (2.0 * M[2]);
  double m = t1;
  int lim = 0;
  if (t2 < m) { m = t2; lim = 1; }
  if (t3 < m) { m = t3; lim = 2; }
  double tau = P.K * m;
  if (P.dt_max < tau) { tau = P.dt_max; lim = 3; }
  if (!isfinite(tau)) {
    C->status = CSPH_EDRY;
    return;
  }
  C->tau = tau;
  C->lim = lim;
  long long k = C->step % LOGCAP;
  dtlog[k] = tau;
  limlog[k] = lim;
}

// Wall ghosts of buffer (parity ^ flip): x-ghosts on owned rows, y-ghosts on
// wall sides (full padded width, so corners are double mirrors).
// Boundary ghosts of buffer (parity ^ flip), DESIGN.md 3.1/3.13: x-ghosts of every padded
// row (wall: mirror, normal momentum negated; open: copy of the boundary cell), then
// y-ghosts over the full padded width on global y edges (corners compose both rules).
template <typename T>
__global__ void mirror_kernel(StripView S, const Ctrl* C, int flip) {
  const int q = C->parity ^ flip;
  if (flip && C->status) return;  // a skipped step leaves the next buffer alone
  T *H = (T*)S.H[q], *Qx = (T*)S.Qx[q], *Qy = (T*)S.Qy[q], *b = (T*)S.b[q];
  const int nx = S.nx, ny = S.ny;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (ny + 2 * GY) * 6) {
    int j = t / 6 - GY, k = t % 6;
    int gi, si;
    bool neg;
    if (k < 3) {
      gi = -1 - k;
      si = S.bc_xlo == 2 ? 0 : k;
      neg = S.bc_xlo == 1;
    } else {
      gi = nx + (k - 3);
      si = S.bc_xhi == 2 ? nx - 1 : nx - 1 - (k - 3);
      neg = S.bc_xhi == 1;
    }
    size_t d = off(S.pitch, gi, j), s = off(S.pitch, si, j);
    H[d] = H[s]; b[d] = b[s]; Qx[d] = neg ? -Qx[s] : Qx[s]; Qy[d] = Qy[s];
  }
}

template <typename T>
__global__ void mirror_y_kernel(StripView S, const Ctrl* C, int flip) {
  const int q = C->parity ^ flip;
  if (flip && C->status) return;
  T *H = (T*)S.H[q], *Qx = (T*)S.Qx[q], *Qy = (T*)S.Qy[q], *b = (T*)S.b[q];
  const int nx = S.nx, ny = S.ny;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int w = nx + 6;
  if (t >= w * 6) return;
  int i = t % w - 3, k = t / w;  // k 0..2: low side, 3..5: high side
  int gj, sj, mode;
  if (k < 3) {
    mode = S.wall_lo;
    gj = -1 - k; sj = mode == 2 ? 0 : k;
  } else {
    mode = S.wall_hi;
    gj = ny + (k - 3); sj = mode == 2 ? ny - 1 : ny - 1 - (k - 3);
  }
  if (!mode) return;
  size_t d = off(S.pitch, i, gj), s = off(S.pitch, i, sj);
  H[d] = H[s]; b[d] = b[s]; Qx[d] = Qx[s]; Qy[d] = mode == 1 ? -Qy[s] : Qy[s];
}

__global__ void w_from_psi_kernel(double* W, const double* psi, size_t n) {  // in place ok
  size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) W[k] = 1.0 / (1.0 - psi[k]);
}

// Step 9 on a freshly set state: maxima over owned wet cells of buffer `parity`.
__global__ void maxima_kernel(StripView S, const Ctrl* C, Phys P, unsigned long long* gM) {
  const int p = C->parity;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  unsigned long long m0 = 0, m1 = 0, m2 = 0;
  if (i < S.nx && j < S.ny) {
    size_t c = off(S.pitch, i, j);
    double H = S.H[p][c];
    if (H > P.eps) {
      double t1, t2, t3;
      dt_terms(P, H, S.Qx[p][c], S.Qy[p][c], S.W ? S.W[c] : S.Wc, cell_aj(P, S, c, H), t1, t2,
               t3);
      m0 = dbits(t1); m1 = dbits(t2); m2 = dbits(t3);
    }
  }
  block_max3_atomic<8>(m0, m1, m2, gM);
}

// NEXT-3: validate the uploaded field rows and turn n_M into c_gam = g n_M^2 in place.
__global__ void fields_kernel(StripView S, double* cg, double* beta, double* src,
                              double* aj0, int jlo, int jhi, double g, double n_scalar,
                              int has_n, int has_b, int has_s, int* flags) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int j = jlo + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  int f = 0;
  if (i < S.nx && j < jhi) {
    size_t c = off(S.pitch, i, j);
    if (cg) {
      double n = has_n ? cg[c] : n_scalar;
      if (!(n >= 0.0 && isfinite(n))) f |= 1;
      cg[c] = g * (n * n);
      if (aj0) aj0[c] = 0.05 * ((n * n) * n);  // Eq.4 numerator
    }
    if (beta) {
      double b = has_b ? beta[c] : 0.0;
      if (!(b >= 0.0 && isfinite(b))) f |= 2;
      beta[c] = b;
      double q = has_s ? src[c] : 0.0;
      if (!(q >= 0.0 && isfinite(q))) f |= 4;
      src[c] = q;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// Boundary ghosts of a static per-cell field (copy: mirror on walls, boundary cell on
// open sides).
__global__ void mirror_field_kernel(StripView S, double* F) {
  const int nx = S.nx, ny = S.ny;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (ny + 2 * GY) * 6) {
    int j = t / 6 - GY, k = t % 6;
    int gi = k < 3 ? -1 - k : nx + (k - 3);
    int si = k < 3 ? (S.bc_xlo == 2 ? 0 : k) : (S.bc_xhi == 2 ? nx - 1 : nx - 1 - (k - 3));
    F[off(S.pitch, gi, j)] = F[off(S.pitch, si, j)];
  }
}

__global__ void mirror_field_y_kernel(StripView S, double* F) {
  const int nx = S.nx, ny = S.ny;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int w = nx + 6;
  if (t >= w * 6) return;
  int i = t % w - 3, k = t / w;
  if (k < 3) {
    if (!S.wall_lo) return;
    F[off(S.pitch, i, -1 - k)] = F[off(S.pitch, i, S.wall_lo == 2 ? 0 : k)];
  } else {
    if (!S.wall_hi) return;
    F[off(S.pitch, i, ny + (k - 3))] =
        F[off(S.pitch, i, S.wall_hi == 2 ? ny - 1 : ny - 1 - (k - 3))];
  }
}

// fp32 state: the same Eq.7 terms computed in fp32 (NEXT-2), maxima kept as fp64 bits.
__global__ void maxima32_kernel(StripView S, const Ctrl* C, Phys P, unsigned long long* gM) {
  const int p = C->parity;
  const PT<float> Q = make_pt<float>(P);
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  unsigned long long m0 = 0, m1 = 0, m2 = 0;
  if (i < S.nx && j < S.ny) {
    size_t c = off(S.pitch, i, j);
    const float H = ((const float*)S.H[p])[c];
    if (H > Q.eps) {
      float t1, t2, t3;
      const float W = S.W ? ((const float*)S.W)[c] : (float)S.Wc;
      dt_terms_t<false>(Q, H, ((const float*)S.Qx[p])[c], ((const float*)S.Qy[p])[c], W, Q.A_J,
                        t1, t2, t3);
      m0 = dbits_t(t1); m1 = dbits_t(t2); m2 = dbits_t(t3);
    }
  }
  block_max3_atomic<8>(m0, m1, m2, gM);
}

// fp64 <-> fp32 conversion of one padded field (NEXT-2 set/get state)
__global__ void to_f32_kernel(float* dst, const double* src, size_t n) {
  size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = (float)src[k];
}
__global__ void to_f64_kernel(double* dst, const float* src, size_t n) {
  size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = (double)src[k];
}

__global__ void max_gather_kernel(unsigned long long* dst, const unsigned long long* src,
                                  int n) {
  if (threadIdx.x < 4) {  // the 3 Eq.7 maxima and the negative-depth flag
    unsigned long long m = 0;
    for (int k = 0; k < n; ++k) {
      unsigned long long v = src[4 * k + threadIdx.x];
      m = v > m ? v : m;
    }
    dst[threadIdx.x] = m;
  }
}

__global__ void init_ctrl_kernel(Ctrl* C) {
  C->tau = 0.0; C->t = 0.0; C->step = 0; C->lim = -1; C->status = 0; C->parity = 0;
}

// Self-test of the branch-free reciprocal / square root against IEEE / and sqrt
// on counter-hashed positive normal inputs with exponents in [-lo, +lo].
__global__ void selftest_math_kernel(long long n, unsigned long long seed, int lo,
                                     unsigned long long* bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long st = (long long)gridDim.x * blockDim.x;
  unsigned long long nb = 0;
  for (; i < n; i += st) {
    unsigned long long z = seed + (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    unsigned long long e = 1023 - lo + (z >> 52) % (2 * lo + 1);
    double x = __longlong_as_double((long long)((e << 52) | (z & 0xFFFFFFFFFFFFFull)));
    if (rcp_nb(x) != 1.0 / x) nb++;
    if (sqrt_nb(x) != sqrt(x)) nb++;
    {  // structured significands: all ones, near all ones, near zero, one bit cleared
      const unsigned long long ONES = 0xFFFFFFFFFFFFFull;
      const unsigned long long k = (unsigned long long)i;
      const unsigned long long ms[3] = {ONES - (k & 255), k & 255, ONES ^ (1ull << (k % 52))};
      for (int q = 0; q < 3; ++q) {
        const double y = __longlong_as_double((long long)((e << 52) | ms[q]));
        if (rcp_nb(y) != 1.0 / y) nb++;
        if (sqrt_nb(y) != sqrt(y)) nb++;
        if (sqrt0nb(y) != sqrt(y)) nb++;
      }
    }
    double t = x * 0x1p-1000;  // tiny and subnormal arguments of sqrt0nb
    if (sqrt0nb(t) != sqrt(t)) nb++;
    if (sqrt0nb(x) != sqrt(x)) nb++;
    if (i == 0) {  // zeros keep their sign; negatives and NaN pass through
      if (__double_as_longlong(sqrt0nb(0.0)) != 0ll) nb++;
      if (__double_as_longlong(sqrt0nb(-0.0)) != __double_as_longlong(-0.0)) nb++;
      if (sqrt0nb(0x1p-1074) != 0x1p-537) nb++;
      if (sqrt0nb(0x1p800) != 0x1p400 || sqrt0nb(0x1.fffffffffffffp799) != sqrt(0x1.fffffffffffffp799)) nb++;
      if (sqrt0nb(0x1p-900) != 0x1p-450 || sqrt0nb(0x1.fffffffffffffp-901) != sqrt(0x1.fffffffffffffp-901)) nb++;
    }
  }
  if (nb) atomicAdd(bad, nb);
}

}  // namespace

namespace ck {
void launch_mirror(const StripView& S, const Ctrl* C, int flip, cudaStream_t st,
                   long long* nlaunch) {
  int n1 = (S.ny + 2 * GY) * 6;
  int n2 = (S.nx + 6) * 6;
  if (S.prec == 4) {
    mirror_kernel<float><<<(n1 + 255) / 256, 256, 0, st>>>(S, C, flip);
    mirror_y_kernel<float><<<(n2 + 255) / 256, 256, 0, st>>>(S, C, flip);
  } else {
    mirror_kernel<double><<<(n1 + 255) / 256, 256, 0, st>>>(S, C, flip);
    mirror_y_kernel<double><<<(n2 + 255) / 256, 256, 0, st>>>(S, C, flip);
  }
  *nlaunch += 2;
}
}  // namespace ck

// ---------------------------------------------------------------- helpers

static Phys make_phys(double dx, const csph_params& p) {
  Phys P{};
  P.g = p.g;
  P.eps = p.eps_dry;
  P.neg_tol = p.neg_tol;
  P.A_J = p.A_J;
  P.C_J = p.C_J;
  P.C_Sh = p.C_Sh;
  double c2 = p.C_Sh * p.C_Sh;
  P.kappa = ((c2 * c2) * c2) * (p.d50 * p.d50);
  P.cP = p.g / (2.0 * dx);
  P.cPh = 0.5 * P.cP;
  P.cgam = p.g * (p.n_manning * p.n_manning);
  P.inv_h = 1.0 / dx;
  P.inv_2h = 1.0 / (2.0 * dx);
  P.h = dx;
  P.K = p.K;
  P.dt_max = p.dt_max;
  P.src = p.q_plus - p.q_minus;
  P.fric = p.n_manning > 0.0;
  P.transport = p.A_J > 0.0 || p.aj_mode == 1;
  P.m_grass = p.m_grass;
  P.m_real = p.m_real;
  P.aj_mode = p.aj_mode;
  P.aj0 = 0.05 * ((p.n_manning * p.n_manning) * p.n_manning);
  P.sm1 = p.s_rel - 1.0;
  P.d50 = p.d50;
  P.hbm = p.h_bed_min < 0.0 ? p.d50 : p.h_bed_min;  // reading #31 film cut-off depth
  return P;
}

static int check_params(int nx, int ny, double dx, const csph_params* p) {
  if (!p) return fail(CSPH_EINVAL, "params is NULL");
  if (nx < 3 || ny < 3) return fail(CSPH_EINVAL, "nx, ny must be >= 3 (got %d, %d)", nx, ny);
  if (!(dx > 0.0) || !std::isfinite(dx)) return fail(CSPH_EINVAL, "dx must be > 0");
  if (!(p->g > 0.0) || !std::isfinite(p->g)) return fail(CSPH_EINVAL, "g must be > 0");
  if (!(p->K > 0.0 && p->K < 1.0)) return fail(CSPH_EINVAL, "K must be in (0,1)");
  if (!(p->eps_dry >= 1e-200) || !(p->eps_dry < 1e200))
    return fail(CSPH_EINVAL, "eps_dry must be in [1e-200, 1e200) (wet depths are divided by)");
  if (!(p->dt_max > 0.0)) return fail(CSPH_EINVAL, "dt_max must be > 0");
  if (!(p->neg_tol >= 0.0)) return fail(CSPH_EINVAL, "neg_tol must be >= 0");
  if (!(p->n_manning >= 0.0) || !std::isfinite(p->n_manning)) return fail(CSPH_EINVAL, "n_manning");
  if (!(p->A_J >= 0.0) || !std::isfinite(p->A_J)) return fail(CSPH_EINVAL, "A_J");
  if (p->m_grass < 0 || p->m_grass > 8) return fail(CSPH_EINVAL, "m_grass must be an integer in 0..8");
  if (p->aj_mode != 0 && p->aj_mode != 1) return fail(CSPH_EINVAL, "aj_mode must be 0 or 1");
  if (p->aj_mode == 1 && !(p->s_rel > 1.0 && std::isfinite(p->s_rel) && p->d50 > 0.0))
    return fail(CSPH_EINVAL, "Eq.4 mode needs s_rel > 1 and d50 > 0");
  if (!std::isfinite(p->C_J)) return fail(CSPH_EINVAL, "C_J");
  if (!(p->C_Sh >= 0.0) || !std::isfinite(p->C_Sh)) return fail(CSPH_EINVAL, "C_Sh");
  if (p->C_Sh > 0.0 && !(p->d50 > 0.0)) return fail(CSPH_EINVAL, "d50 must be > 0 when C_Sh > 0");
  if (!std::isfinite(p->q_plus) || !std::isfinite(p->q_minus)) return fail(CSPH_EINVAL, "q_plus/q_minus");
  if (p->precision != 64 && p->precision != 32) return fail(CSPH_EINVAL, "precision must be 64 or 32");
  if (p->precision == 32 && (p->path != CSPH_PATH_FUSED || p->m_grass != 2 || p->aj_mode != 0 ||
                             p->open_bc != 0))
    return fail(CSPH_EINVAL,
                "precision 32 (NEXT-2) runs the fused path with walls, m_grass = 2, constant A_J");
  if (p->path != CSPH_PATH_FUSED && p->path != CSPH_PATH_STAGED) return fail(CSPH_EINVAL, "path");
  if (p->open_bc < 0 || p->open_bc > 15) return fail(CSPH_EINVAL, "open_bc is a 4-bit mask");
  if (std::isnan(p->h_bed_min) || !(p->h_bed_min < INFINITY))
    return fail(CSPH_EINVAL, "h_bed_min must be finite (< 0 selects d50)");
  if (!(p->m_real < 0.0) && !(p->m_real >= 0.0 && p->m_real <= 8.0))
    return fail(CSPH_EINVAL, "m_real must be in [0, 8] (or < 0: use m_grass)");
  if (p->precision == 32 && p->m_real >= 0.0)
    return fail(CSPH_EINVAL, "m_real (pinned pow) is fp64 only");
  return CSPH_OK;
}

static int dalloc(Strip& s, void** ptr, size_t bytes) {
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return fail(CSPH_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  }
  s.allocs.push_back(*ptr);
  return CSPH_OK;
}

static int strip_init(csph* H, Strip& s, int dev, int gj0, int rows, bool staged) {
  s.dev = dev;
  s.gj0 = gj0;
  CK(cudaSetDevice(dev));
  StripView& v = s.v;
  v.nx = H->nx;
  v.ny = rows;
  // padded row: GX left + nx + 3 right ghosts, plus slack so that the fused kernel's TMA row
  // copies (rounded up to 16 B: up to 3 fp32 / 1 fp64 element past the last ghost) stay
  // inside the row; rounded up to 32 elements (256 B)
  v.pitch = ((H->nx + GX + 3 + 4) + 31) / 32 * 32;
  // y edges: 0 halo (interior strip edge), 1 wall, 2 open; x edges: 1 wall, 2 open
  const int ob = H->p.open_bc;
  v.wall_lo = gj0 == 0 ? ((ob & 4) ? 2 : 1) : 0;
  v.wall_hi = gj0 + rows == H->ny ? ((ob & 8) ? 2 : 1) : 0;
  v.bc_xlo = (ob & 1) ? 2 : 1;
  v.bc_xhi = (ob & 2) ? 2 : 1;
  v.prec = H->p.precision == 32 ? 4 : 8;
  v.W = nullptr;
  v.Wc = 1.0;
  size_t n = (size_t)(rows + 2 * GY) * v.pitch;
  int st;
  for (int k = 0; k < 2; ++k) {
    if ((st = dalloc(s, (void**)&v.H[k], n * 8))) return st;
    if ((st = dalloc(s, (void**)&v.Qx[k], n * 8))) return st;
    if ((st = dalloc(s, (void**)&v.Qy[k], n * 8))) return st;
    if ((st = dalloc(s, (void**)&v.b[k], n * 8))) return st;
    CK(cudaMemset(v.H[k], 0, n * 8));
    CK(cudaMemset(v.Qx[k], 0, n * 8));
    CK(cudaMemset(v.Qy[k], 0, n * 8));
    CK(cudaMemset(v.b[k], 0, n * 8));
  }
  if ((st = dalloc(s, (void**)&s.ctrl, sizeof(Ctrl)))) return st;
  CK(cudaMemset(s.ctrl, 0, sizeof(Ctrl)));  // padding bytes too (they travel to the host)
  if ((st = dalloc(s, (void**)&s.gM, 4 * sizeof(unsigned long long)))) return st;
  if ((st = dalloc(s, (void**)&s.Mlast, 4 * sizeof(double)))) return st;
  if ((st = dalloc(s, (void**)&s.dtlog, LOGCAP * sizeof(double)))) return st;
  if ((st = dalloc(s, (void**)&s.limlog, LOGCAP * sizeof(int)))) return st;
  if ((st = dalloc(s, (void**)&s.dflags, 4 * sizeof(int)))) return st;
  {
    // tile rows: the caller's, or chosen from the state at every set_state (tile_rows_auto);
    // until then 128.  The flag buffers are sized for the finest tiling (16 rows).
    s.ntx = (v.nx + FUSED_TX - 1) / FUSED_TX;
    s.auto_ty = H->p.tile_rows <= 0;
    s.ty = s.auto_ty ? 128 : H->p.tile_rows;
    s.nty = (v.ny + s.ty - 1) / s.ty;
    const int tymin = s.auto_ty ? kTyMin : s.ty;
    const size_t nt = (size_t)s.ntx * ((v.ny + tymin - 1) / tymin);
    if ((st = dalloc(s, (void**)&s.tflag, 2 * nt))) return st;
    if ((st = dalloc(s, (void**)&s.tstate, nt))) return st;
    if ((st = dalloc(s, (void**)&s.gflag, 4 * (size_t)s.ntx))) return st;
    CK(cudaMemset(s.gflag, HGS_ALL, 4 * (size_t)s.ntx));
    s.tflag_cap = nt;
    CK(cudaMemset(s.tflag, HGS_ALL, 2 * nt));
    CK(cudaMemset(s.tstate, 0, nt));
    if (s.auto_ty) {
      if ((st = dalloc(s, (void**)&s.wetblk, nt))) return st;
      CK(cudaDeviceGetAttribute(&s.nsm, cudaDevAttrMultiProcessorCount, s.dev));
    }
    if ((st = dalloc(s, (void**)&s.hstats, 4 * sizeof(unsigned long long)))) return st;
    CK(cudaMemset(s.hstats, 0, 4 * sizeof(unsigned long long)));
    if ((st = dalloc(s, (void**)&s.tcost, 2 * nt * sizeof(unsigned short)))) return st;
    if ((st = dalloc(s, (void**)&s.torder, 2 * nt * sizeof(int)))) return st;
  }
  CK(cudaMemset(s.gM, 0, 4 * sizeof(unsigned long long)));
  CK(cudaMemset(s.Mlast, 0, 4 * sizeof(double)));
  if (staged) {
    Scratch& T = s.scr;
    double** arr[] = {&T.eta, &T.r, &T.u, &T.v, &T.phix, &T.phiy, &T.gam, &T.Hh, &T.ut,
                      &T.vt, &T.phix2, &T.phiy2, &T.QLx, &T.QLy, &T.J0x, &T.J0y, &T.J0a,
                      &T.FH, &T.FQx, &T.FQy, &T.FJ, &T.GH, &T.GQx, &T.GQy, &T.GJ};
    for (auto a : arr) {
      if ((st = dalloc(s, (void**)a, n * 8))) return st;
      CK(cudaMemset(*a, 0, n * 8));
    }
    if ((st = dalloc(s, (void**)&T.w, n))) return st;
    CK(cudaMemset(T.w, 0, n));
    s.has_scr = true;
  }
  CK(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
  s.own_stream = true;
  CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&s.cst, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&s.ev_edge, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_int, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_comm, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&s.ost, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&s.ev_ofork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_ojoin, cudaEventDisableTiming));
  init_ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s.st));
  return CSPH_OK;
}

static void strip_free(Strip& s) {
  cudaSetDevice(s.dev);
  if (s.sst) cudaStreamSynchronize(s.sst);  // a pending asynchronous Save reads s.snap
  if (s.ost) cudaStreamSynchronize(s.ost);
  if (s.st) cudaStreamSynchronize(s.st);
  for (void* p : s.allocs) cudaFree(p);
  s.allocs.clear();
  if (s.st && s.own_stream) cudaStreamDestroy(s.st);
  if (s.ev) cudaEventDestroy(s.ev);
  if (s.cst) {
    cudaStreamSynchronize(s.cst);
    cudaStreamDestroy(s.cst);
  }
  if (s.ost) cudaStreamDestroy(s.ost);
  if (s.sst) cudaStreamDestroy(s.sst);
  for (cudaEvent_t e : {s.ev_edge, s.ev_int, s.ev_comm, s.ev_ofork, s.ev_ojoin, s.ev_snap,
                        s.ev_saved})
    if (e) cudaEventDestroy(e);
  s.sst = nullptr;
  s.ev_snap = s.ev_saved = nullptr;
  s.snap = nullptr;
  s.save_issued = false;
  s.ost = nullptr;
  s.cst = nullptr;
  s.st = nullptr;
  s.ev = nullptr;
}

namespace {
// Wet flags of the 120-column x kTyMin-row blocks of the current state (buffer 0).
template <typename T>
__global__ void wet_blocks_kernel(StripView S, double eps, unsigned char* out, int buf) {
  const int bx = blockIdx.x, by = blockIdx.y, t = threadIdx.x;
  const int col = bx * FUSED_TX + t;
  const T* H = reinterpret_cast<const T*>(S.H[buf]);
  bool wet = false;
  if (t < FUSED_TX && col < S.nx) {
    const int j1 = min(S.ny, (by + 1) * kTyMin);
    for (int j = by * kTyMin; j < j1; ++j) wet |= (double)H[off(S.pitch, col, j)] > eps;
  }
  wet = __syncthreads_or(wet);
  if (t == 0) out[by * gridDim.x + bx] = wet ? 1 : 0;
}

// Wet cells per owned row of buffer `buf` (one block per row): the cost model of the row-strip
// partition.
template <typename T>
__global__ void row_wet_kernel(StripView S, double eps, int buf, int* out) {
  const int j = blockIdx.x;
  const T* H = reinterpret_cast<const T*>(S.H[buf]);
  int n = 0;
  for (int i = threadIdx.x; i < S.nx; i += blockDim.x) n += (double)H[off(S.pitch, i, j)] > eps;
  n = __reduce_add_sync(0xffffffffu, n);
  __shared__ int part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    out[j] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------- C-ABI

extern "C" {

void csph_default_params(csph_params* p) {
  if (!p) return;
  p->g = 9.81;
  p->K = 0.25;
  p->eps_dry = 1e-6;
  p->dt_max = INFINITY;
  p->neg_tol = 1e-12;
  p->n_manning = 0.0;
  p->A_J = 0.0;
  p->m_grass = 2;
  p->C_J = 0.0;
  p->C_Sh = 0.0;
  p->d50 = 1e-3;
  p->q_plus = 0.0;
  p->q_minus = 0.0;
  p->precision = 64;
  p->device = 0;
  p->path = CSPH_PATH_FUSED;
  p->tile_rows = 0;
  p->hgs = 1;
  p->aj_mode = 0;
  p->s_rel = 2.65;
  p->open_bc = 0;
  p->graphs = 1;
  p->h_bed_min = -1.0;
  p->halo_push = 1;
  p->m_real = -1.0;
}

const char* csph_last_error(void) { return g_err.c_str(); }

const char* csph_strerror(int code) {
  switch (code) {
    case CSPH_OK: return "ok";
    case CSPH_EINVAL: return "invalid argument";
    case CSPH_ENOSTATE: return "no state (call csph_set_state first)";
    case CSPH_ENOMEM: return "device out of memory";
    case CSPH_ECUDA: return "CUDA error";
    case CSPH_ENCCL: return "NCCL error";
    case CSPH_ENEGDEPTH: return "negative depth below -neg_tol";
    case CSPH_ENONFINITE: return "non-finite Eq.7 maximum";
    case CSPH_EDRY: return "no wet cell and dt_max = inf";
    default: return "unknown error";
  }
}

int csph_strip_rows(int ny, int nranks, int rank, int* j0, int* j1) {
  if (nranks < 1 || rank < 0 || rank >= nranks || ny < 3)
    return fail(CSPH_EINVAL, "bad strip request");
  int base = ny / nranks, extra = ny % nranks;
  int a = rank * base + (rank < extra ? rank : extra);
  int n = base + (rank < extra ? 1 : 0);
  if (n < GY) return fail(CSPH_EINVAL, "strip of %d rows < %d (too many ranks for ny=%d)", n, GY, ny);
  if (j0) *j0 = a;
  if (j1) *j1 = a + n;
  return CSPH_OK;
}

static csph* make_handle(int nx, int ny, double dx, const csph_params* p) {
  if (check_params(nx, ny, dx, p)) return nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) {
    fail(CSPH_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
    return nullptr;
  }
  csph* H = new csph();
  H->nx = nx;
  H->ny = ny;
  H->dx = dx;
  H->p = *p;
  H->P = make_phys(dx, *p);
  H->graphs = p->graphs != 0;
  return H;
}

csph_t* csph_create(int nx, int ny, double dx, const csph_params* p) {
  csph* H = make_handle(nx, ny, dx, p);
  if (!H) return nullptr;
  H->mode = SINGLE;
  H->s.resize(1);
  if (strip_init(H, H->s[0], p->device, 0, ny, p->path == CSPH_PATH_STAGED)) {
    std::string keep = g_err;
    csph_destroy(H);
    g_err = keep;
    return nullptr;
  }
  return H;
}

// bounds[0..n]: 0 = bounds[0] < ... < bounds[n] = ny, every strip >= GY rows
static int check_bounds(int ny, int n, const int* bounds) {
  if (!bounds) return fail(CSPH_EINVAL, "bounds is NULL");
  if (bounds[0] != 0 || bounds[n] != ny) return fail(CSPH_EINVAL, "bounds must run from 0 to ny");
  for (int r = 0; r < n; ++r)
    if (bounds[r + 1] - bounds[r] < GY)
      return fail(CSPH_EINVAL, "strip %d has %d rows (< %d)", r, bounds[r + 1] - bounds[r], GY);
  return CSPH_OK;
}

static int even_bounds(int ny, int n, std::vector<int>& b) {
  b.assign(n + 1, 0);
  for (int r = 0; r < n; ++r) {
    int st = csph_strip_rows(ny, n, r, &b[r], &b[r + 1]);
    if (st) return st;
  }
  return CSPH_OK;
}

int csph_balance_rows(int ny, int nranks, const double* w, int* bounds) {
  if (ny < GY || nranks < 1 || !w || !bounds || (long long)nranks * GY > ny)
    return fail(CSPH_EINVAL, "bad balance request (ny=%d, nranks=%d)", ny, nranks);
  double tot = 0.0;
  for (int j = 0; j < ny; ++j) {
    if (!(w[j] >= 0.0) || !std::isfinite(w[j])) return fail(CSPH_EINVAL, "row weight %d invalid", j);
    tot += w[j];
  }
  std::vector<int> b;
  if (!(tot > 0.0)) {  // nothing to balance: the even split
    int st = even_bounds(ny, nranks, b);
    if (st) return st;
    for (int r = 0; r <= nranks; ++r) bounds[r] = b[r];
    return CSPH_OK;
  }
  // feasible(T): can rows [0, ny) be cut into nranks contiguous strips of >= GY rows, each
  // of cost <= T?  reach[r][e] = rows [0, e) split into r such strips; the best start for
  // an end e is the largest reachable s <= e - GY (costs are >= 0).  O(nranks * ny).
  std::vector<double> pre(ny + 1, 0.0);
  for (int j = 0; j < ny; ++j) pre[j + 1] = pre[j] + w[j];
  std::vector<std::vector<char>> reach(nranks + 1, std::vector<char>(ny + 1, 0));
  auto feasible = [&](double T) {
    for (auto& v : reach) std::fill(v.begin(), v.end(), 0);
    reach[0][0] = 1;
    for (int r = 1; r <= nranks; ++r) {
      int last = -1;
      for (int e = GY; e <= ny; ++e) {
        if (reach[r - 1][e - GY]) last = e - GY;
        if (last >= 0 && pre[e] - pre[last] <= T) reach[r][e] = 1;
      }
    }
    return reach[nranks][ny] != 0;
  };
  // bisection on the largest strip cost T, then walk the cuts back from ny
  double lo = 0.0, hi = tot;
  for (int it = 0; it < 200 && hi - lo > 1e-13 * hi; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (feasible(mid)) hi = mid; else lo = mid;
  }
  if (!feasible(hi)) return fail(CSPH_EINVAL, "no partition of %d rows into %d strips", ny, nranks);
  b.assign(nranks + 1, 0);
  b[nranks] = ny;
  for (int r = nranks; r >= 1; --r) {
    const int e = b[r];
    int s0 = e - GY;
    while (s0 >= 0 && !(reach[r - 1][s0] && pre[e] - pre[s0] <= hi)) --s0;
    if (s0 < 0) return fail(CSPH_EINVAL, "partition walk-back failed");
    b[r - 1] = s0;
  }
  for (int r = 0; r <= nranks; ++r) bounds[r] = b[r];
  return check_bounds(ny, nranks, bounds);
}

// ---- halo push: the neighbours' buffers a strip's step kernel writes into

static void push_clear(StripView& v) {
  for (int side = 0; side < 2; ++side) {
    for (int k = 0; k < 2; ++k) v.nH[side][k] = v.nQx[side][k] = v.nQy[side][k] = v.nb[side][k] = nullptr;
    v.ndel[side] = 0;
    v.ngflag[side] = nullptr;
  }
}

// Side `side` of v pushes into the buffers Hs..bs[2] and ghost flags gflag of the neighbour;
// del: element offset from v's (col, j) to the neighbour's copy of that cell.
static void push_side(StripView& v, int side, double* const Hs[2], double* const Qxs[2],
                      double* const Qys[2], double* const bs[2], unsigned char* gflag,
                      long long del) {
  for (int k = 0; k < 2; ++k) {
    v.nH[side][k] = Hs[k];
    v.nQx[side][k] = Qxs[k];
    v.nQy[side][k] = Qys[k];
    v.nb[side][k] = bs[k];
  }
  v.ndel[side] = del;
  v.ngflag[side] = gflag;
}

// The peer combine's inbox of a strip for nranks ranks (zeroed) and its device array of the
// ranks' inbox pointers (peers[r], host array of nranks).
static int combine_alloc(Strip& s, int nranks) {
  CK(cudaSetDevice(s.dev));
  const size_t nb = 2 * (size_t)nranks * kInboxW * sizeof(unsigned long long);
  int st;
  if (!s.inbox) {
    if ((st = dalloc(s, (void**)&s.inbox, nb))) return st;
    if ((st = dalloc(s, (void**)&s.dpeers, (size_t)nranks * sizeof(void*)))) return st;
  }
  CK(cudaMemset(s.inbox, 0, nb));
  return CSPH_OK;
}

static int combine_set_peers(Strip& s, const std::vector<unsigned long long*>& peers) {
  CK(cudaSetDevice(s.dev));
  CK(cudaMemcpy(s.dpeers, peers.data(), peers.size() * sizeof(void*), cudaMemcpyHostToDevice));
  return CSPH_OK;
}

// The ctrl kernel's combine arguments for strip r (none unless the peers are linked).
static PeerCombine combine_of(const csph* H, const Strip& s, int r) {
  PeerCombine pc{};
  if (H->p2p_combine) {
    pc.peers = s.dpeers;
    pc.inbox = s.inbox;
    pc.nranks = H->nranks;
    pc.rank = r;
  }
  return pc;
}

// MULTI: strip r pushes its rows 0..2 into the upper ghost rows of strip r-1 and its rows
// ny-3..ny-1 into the lower ghost rows of strip r+1 (same device, or peer access between
// the devices); otherwise (or halo_push = 0, or the staged path) the peer copies stay.
static void push_link_multi(csph* H) {
  H->push = false;
  H->p2p_combine = false;
  for (auto& s : H->s) push_clear(s.v);
  const int n = (int)H->s.size();
  if (!H->p.halo_push || H->p.path != CSPH_PATH_FUSED) return;
  if (n < 2) {  // no interior edge: nothing to push, the strip is launched whole
    H->push = true;
    return;
  }
  for (int r = 0; r + 1 < n; ++r) {
    const int a = H->s[r].dev, b = H->s[r + 1].dev;
    int ab = 1, ba = 1;
    if (a != b) {
      cudaDeviceCanAccessPeer(&ab, a, b);
      cudaDeviceCanAccessPeer(&ba, b, a);
    }
    if (!ab || !ba) return;
  }
  for (int r = 0; r < n; ++r) {
    StripView& v = H->s[r].v;
    if (r > 0) {
      Strip& o = H->s[r - 1];
      push_side(v, 0, o.v.H, o.v.Qx, o.v.Qy, o.v.b, o.gflag, (long long)o.v.ny * v.pitch);
    }
    if (r < n - 1) {
      Strip& o = H->s[r + 1];
      push_side(v, 1, o.v.H, o.v.Qx, o.v.Qy, o.v.b, o.gflag, -(long long)v.ny * v.pitch);
    }
  }
  H->push = true;
  // and the maxima combined by the ctrl kernels through every strip's inbox
  std::vector<unsigned long long*> peers;
  for (auto& s : H->s) {
    if (combine_alloc(s, n)) return;
    peers.push_back(s.inbox);
  }
  for (auto& s : H->s)
    if (combine_set_peers(s, peers)) return;
  H->p2p_combine = true;
}

csph_t* csph_create_multi(int nx, int ny, double dx, const csph_params* p, int nstrips,
                          const int* devices) {
  std::vector<int> b;
  if (nstrips < 1 || even_bounds(ny, nstrips, b)) {
    if (nstrips < 1) fail(CSPH_EINVAL, "nstrips < 1");
    return nullptr;
  }
  return csph_create_multi_rows(nx, ny, dx, p, nstrips, devices, b.data());
}

csph_t* csph_create_multi_rows(int nx, int ny, double dx, const csph_params* p, int nstrips,
                               const int* devices, const int* bounds) {
  if (nstrips < 1 || !devices) {
    fail(CSPH_EINVAL, "nstrips < 1 or devices NULL");
    return nullptr;
  }
  if (check_bounds(ny, nstrips, bounds)) return nullptr;
  csph* H = make_handle(nx, ny, dx, p);
  if (!H) return nullptr;
  H->mode = MULTI;
  H->nranks = nstrips;
  H->s.resize(nstrips);
  for (int r = 0; r < nstrips; ++r) {
    const int j0 = bounds[r], j1 = bounds[r + 1];
    if (strip_init(H, H->s[r], devices[r], j0, j1 - j0, p->path == CSPH_PATH_STAGED)) {
      std::string keep = g_err;
      csph_destroy(H);
      g_err = keep;
      return nullptr;
    }
  }
  // peer access where devices differ (ignore "already enabled")
  for (int a = 0; a < nstrips; ++a)
    for (int b = 0; b < nstrips; ++b)
      if (H->s[a].dev != H->s[b].dev) {
        cudaSetDevice(H->s[a].dev);
        cudaDeviceEnablePeerAccess(H->s[b].dev, 0);
        cudaGetLastError();
      }
  cudaSetDevice(H->s[0].dev);
  if (cudaMalloc((void**)&H->gather, (size_t)nstrips * 4 * sizeof(unsigned long long)) !=
      cudaSuccess) {
    fail(CSPH_ENOMEM, "gather buffer");
    csph_destroy(H);
    return nullptr;
  }
  push_link_multi(H);
  return H;
}

int csph_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int csph_make_nccl_id(void* out) {
  if (!out) return fail(CSPH_EINVAL, "out is NULL");
  if (!load_nccl()) return CSPH_ENCCL;
  ncclUniqueId id;
  NK(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return CSPH_OK;
}

csph_t* csph_create_dist(int nx, int ny, double dx, const csph_params* p, int rank,
                         int nranks, int local_device, const void* nccl_id) {
  std::vector<int> b;
  if (nranks < 1 || even_bounds(ny, nranks, b)) {
    if (nranks < 1) fail(CSPH_EINVAL, "nranks < 1");
    return nullptr;
  }
  return csph_create_dist_rows(nx, ny, dx, p, rank, nranks, b.data(), local_device, nccl_id);
}

csph_t* csph_create_dist_rows(int nx, int ny, double dx, const csph_params* p, int rank,
                              int nranks, const int* bounds, int local_device,
                              const void* nccl_id) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !nccl_id) {
    fail(CSPH_EINVAL, "bad rank/nranks/nccl_id");
    return nullptr;
  }
  if (check_bounds(ny, nranks, bounds)) return nullptr;
  const int j0 = bounds[rank], j1 = bounds[rank + 1];
  if (!load_nccl()) return nullptr;
  csph* H = make_handle(nx, ny, dx, p);
  if (!H) return nullptr;
  H->mode = DIST;
  H->rank = rank;
  H->nranks = nranks;
  H->bounds.assign(bounds, bounds + nranks + 1);
  H->s.resize(1);
  if (strip_init(H, H->s[0], local_device, j0, j1 - j0, p->path == CSPH_PATH_STAGED)) {
    std::string keep = g_err;
    csph_destroy(H);
    g_err = keep;
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof id);
  cudaSetDevice(local_device);
  ncclResult_t r = g_nccl.CommInitRank(&H->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    fail(CSPH_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    H->comm = nullptr;
    std::string keep = g_err;
    csph_destroy(H);
    g_err = keep;
    return nullptr;
  }
  // one rank has no interior edge (launched whole); more push once csph_ipc_link has
  // mapped the neighbours' buffers, and send/recv halos until then
  H->push = nranks == 1 && p->halo_push && p->path == CSPH_PATH_FUSED;
  return H;
}

// ---- DIST halo push through CUDA IPC

namespace {
struct IpcBlob {
  int magic, rank, nranks, ny, pitch, ntx, prec;
  cudaIpcMemHandle_t f[4][2];  // H, Qx, Qy, b x parity
  cudaIpcMemHandle_t gflag;
  cudaIpcMemHandle_t inbox;    // the peer combine's inbox
};
constexpr int kIpcMagic = 0x43535048;  // "CSPH"
}  // namespace

static void ipc_unlink(csph* H) {
  for (void* p : H->ipc_open) cudaIpcCloseMemHandle(p);
  H->ipc_open.clear();
  H->p2p_combine = false;
  for (auto& s : H->s) push_clear(s.v);
  H->push = H->mode == DIST && H->nranks == 1 && H->p.halo_push && H->p.path == CSPH_PATH_FUSED;
}

int csph_ipc_blob_bytes(void) { return (int)sizeof(IpcBlob); }

int csph_ipc_export(csph_t* H, void* out) {
  if (!H || !out) return fail(CSPH_EINVAL, "NULL argument");
  if (H->mode != DIST) return fail(CSPH_EINVAL, "csph_ipc_export needs a DIST handle");
  Strip& s = H->s[0];
  CK(cudaSetDevice(s.dev));
  IpcBlob b;
  memset(&b, 0, sizeof b);
  b.magic = kIpcMagic;
  b.rank = H->rank;
  b.nranks = H->nranks;
  b.ny = s.v.ny;
  b.pitch = s.v.pitch;
  b.ntx = s.ntx;
  b.prec = s.v.prec;
  double* const* F[4] = {s.v.H, s.v.Qx, s.v.Qy, s.v.b};
  for (int k = 0; k < 4; ++k)
    for (int q = 0; q < 2; ++q) CK(cudaIpcGetMemHandle(&b.f[k][q], F[k][q]));
  CK(cudaIpcGetMemHandle(&b.gflag, s.gflag));
  int st;
  if ((st = combine_alloc(s, H->nranks))) return st;
  CK(cudaIpcGetMemHandle(&b.inbox, s.inbox));
  memcpy(out, &b, sizeof b);
  return CSPH_OK;
}

static int ipc_open(csph* H, const cudaIpcMemHandle_t& h, void** p) {
  const cudaError_t e = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(CSPH_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  H->ipc_open.push_back(*p);
  return CSPH_OK;
}

int csph_ipc_link(csph_t* H, const void* blobs, int nblobs) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (H->mode != DIST) return fail(CSPH_EINVAL, "csph_ipc_link needs a DIST handle");
  Strip& s = H->s[0];
  CK(cudaSetDevice(s.dev));
  graphs_reset(H);  // captured steps bake in the transports
  ipc_unlink(H);
  if (!blobs && nblobs == 0) return CSPH_OK;  // unlink: send/recv halos, NCCL allreduce
  if (!blobs || nblobs != H->nranks)
    return fail(CSPH_EINVAL, "csph_ipc_link: give every rank's blob (%d), rank order", H->nranks);
  if (!H->p.halo_push || H->p.path != CSPH_PATH_FUSED) return CSPH_OK;
  std::vector<IpcBlob> B(nblobs);
  for (int r = 0; r < nblobs; ++r) {
    memcpy(&B[r], (const char*)blobs + (size_t)r * sizeof(IpcBlob), sizeof(IpcBlob));
    const IpcBlob& b = B[r];
    if (b.magic != kIpcMagic || b.rank != r || b.nranks != H->nranks || b.pitch != s.v.pitch ||
        b.ntx != s.ntx || b.prec != s.v.prec || b.ny != H->bounds[r + 1] - H->bounds[r])
      return fail(CSPH_EINVAL, "csph_ipc_link: blob %d is not rank %d's strip", r, r);
  }
  if (H->nranks == 1) return CSPH_OK;  // no neighbour, nothing to combine across
  int st;
  // halo push: the neighbours' state buffers and ghost-flag rows
  for (int side = 0; side < 2; ++side) {
    const int o = H->rank + (side == 0 ? -1 : 1);
    if (o < 0 || o >= H->nranks) continue;
    double* Fs[4][2];
    for (int k = 0; k < 4; ++k)
      for (int q = 0; q < 2; ++q) {
        void* p = nullptr;
        if ((st = ipc_open(H, B[o].f[k][q], &p))) { ipc_unlink(H); return st; }
        Fs[k][q] = (double*)p;
      }
    void* gf = nullptr;
    if ((st = ipc_open(H, B[o].gflag, &gf))) { ipc_unlink(H); return st; }
    const long long del = side == 0 ? (long long)B[o].ny * s.v.pitch : -(long long)s.v.ny * s.v.pitch;
    push_side(s.v, side, Fs[0], Fs[1], Fs[2], Fs[3], (unsigned char*)gf, del);
  }
  // peer combine: every rank's inbox (mine is local memory)
  if ((st = combine_alloc(s, H->nranks))) { ipc_unlink(H); return st; }
  std::vector<unsigned long long*> peers(H->nranks, nullptr);
  for (int r = 0; r < H->nranks; ++r) {
    if (r == H->rank) { peers[r] = s.inbox; continue; }
    void* p = nullptr;
    if ((st = ipc_open(H, B[r].inbox, &p))) { ipc_unlink(H); return st; }
    peers[r] = (unsigned long long*)p;
  }
  if ((st = combine_set_peers(s, peers))) { ipc_unlink(H); return st; }
  H->push = true;
  H->p2p_combine = true;
  return CSPH_OK;
}

void csph_destroy(csph_t* H) {
  if (!H) return;
  if (!H->s.empty()) cudaSetDevice(H->s[0].dev);
  graphs_free(H);
  for (auto e : H->evs) cudaEventDestroy(e);
  for (void* p : H->ipc_open) cudaIpcCloseMemHandle(p);
  for (auto& s : H->s) strip_free(s);
  if (H->gather) {
    cudaSetDevice(H->s.empty() ? 0 : H->s[0].dev);
    cudaFree(H->gather);
  }
  if (H->comm && g_nccl.ok) g_nccl.CommDestroy(H->comm);
  delete H;
}

int csph_set_stream(csph_t* H, void* stream) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (H->s.size() != 1) return fail(CSPH_EINVAL, "set_stream needs a single-strip handle");
  Strip& s = H->s[0];
  CK(cudaSetDevice(s.dev));
  CK(cudaStreamSynchronize(s.st));
  if (s.own_stream) cudaStreamDestroy(s.st);
  s.st = (cudaStream_t)stream;
  s.own_stream = false;
  return CSPH_OK;
}

long long csph_last_launch_count(csph_t* H) { return H ? H->launches : 0; }

int csph_selftest_math(long long n, unsigned long long seed, long long* mismatches) {
  if (n < 0 || !mismatches) return fail(CSPH_EINVAL, "bad argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return fail(CSPH_ECUDA, "no CUDA device");
  unsigned long long* d = nullptr;
  CK(cudaMalloc((void**)&d, 8));
  CK(cudaMemset(d, 0, 8));
  selftest_math_kernel<<<1024, 256>>>(n, seed, 300, d);
  CK(cudaGetLastError());
  unsigned long long h = 0;
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  CK(cudaFree(d));
  *mismatches = (long long)h;
  return CSPH_OK;
}

int csph_get_tile_stats(csph_t* H, long long counts[3]) {
  if (!H || !counts) return fail(CSPH_EINVAL, "bad argument");
  counts[0] = counts[1] = counts[2] = 0;
  for (auto& s : H->s) {
    unsigned long long c[4];
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.st));
    CK(cudaMemcpy(c, s.hstats, sizeof c, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 3; ++k) counts[k] += (long long)c[k];
  }
  return CSPH_OK;
}

int csph_reset_tile_stats(csph_t* H) {
  if (!H) return fail(CSPH_EINVAL, "bad argument");
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    CK(cudaMemsetAsync(s.hstats, 0, 4 * sizeof(unsigned long long), s.st));
  }
  return CSPH_OK;
}

int csph_profile(csph_t* H, int enable) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  H->profiling = enable != 0;
  H->prof_ms = 0.0;
  H->prof_steps = 0;
  return CSPH_OK;
}

int csph_get_profile(csph_t* H, double* ms, long long* steps) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (ms) *ms = H->prof_ms;
  if (steps) *steps = H->prof_steps;
  return CSPH_OK;
}

// -------- collective pieces of a step

// Where the halo of a strip lives (one place for the NCCL and the peer-copy transports,
// so the multi-strip tests on one GPU exercise the offsets the NCCL path uses).
// State rows, in elements of the padded layout, full padded width from column -GX (so the
// x-ghosts travel too): the 3 owned rows sent to the neighbour below (send_lo, rows
// 0..2) or above (send_hi, rows ny-3..ny-1) and the 3 ghost rows received from it
// (recv_lo, rows -3..-1; recv_hi, rows ny..ny+2).  HGS tile flags of parity q: my first
// tile row goes below, my last above; the neighbours' facing rows land in gflag.
struct HaloMap {
  size_t count;  // elements per field and side
  size_t send_lo, recv_lo, send_hi, recv_hi;
  size_t fsend_lo, fsend_hi;  // into s.tflag
  size_t frecv_lo, frecv_hi;  // into s.gflag
};

static HaloMap halo_map(const Strip& s, int q) {
  const StripView& v = s.v;
  HaloMap m;
  m.count = (size_t)GY * v.pitch;
  m.send_lo = off(v.pitch, -GX, 0);
  m.recv_lo = off(v.pitch, -GX, -GY);
  m.send_hi = off(v.pitch, -GX, v.ny - GY);
  m.recv_hi = off(v.pitch, -GX, v.ny);
  const size_t nt = (size_t)s.ntx * s.nty;
  m.fsend_lo = nt * (size_t)q;
  m.fsend_hi = nt * (size_t)q + (size_t)(s.nty - 1) * s.ntx;
  m.frecv_lo = 2 * (size_t)s.ntx * (size_t)q;
  m.frecv_hi = m.frecv_lo + s.ntx;
  return m;
}

static void state_fields(const StripView& v, int q, char* f[4]) {
  f[0] = (char*)v.H[q]; f[1] = (char*)v.Qx[q]; f[2] = (char*)v.Qy[q]; f[3] = (char*)v.b[q];
}

// NCCL halo exchange of buffer q with ranks r-1 / r+1 (no wrap-around, reading #18).
static int halo_nccl(csph* H, int q, cudaStream_t stream) {
  if (H->nranks == 1) return CSPH_OK;
  Strip& s = H->s[0];
  const StripView& v = s.v;
  const HaloMap m = halo_map(s, q);
  const size_t es = (size_t)v.prec;  // element size: fp64 or fp32 state
  const ncclDataType_t dt = v.prec == 4 ? ncclFloat32 : ncclFloat64;
  char* f[4];
  state_fields(v, q, f);
  const bool lo = H->rank > 0, hi = H->rank < H->nranks - 1;
  NK(g_nccl.GroupStart());
  if (lo) {
    NK(g_nccl.Send(s.tflag + m.fsend_lo, s.ntx, ncclUint8, H->rank - 1, H->comm, stream));
    NK(g_nccl.Recv(s.gflag + m.frecv_lo, s.ntx, ncclUint8, H->rank - 1, H->comm, stream));
  }
  if (hi) {
    NK(g_nccl.Send(s.tflag + m.fsend_hi, s.ntx, ncclUint8, H->rank + 1, H->comm, stream));
    NK(g_nccl.Recv(s.gflag + m.frecv_hi, s.ntx, ncclUint8, H->rank + 1, H->comm, stream));
  }
  for (int k = 0; k < 4; ++k) {
    if (lo) {
      NK(g_nccl.Send(f[k] + es * m.send_lo, m.count, dt, H->rank - 1, H->comm, stream));
      NK(g_nccl.Recv(f[k] + es * m.recv_lo, m.count, dt, H->rank - 1, H->comm, stream));
    }
    if (hi) {
      NK(g_nccl.Send(f[k] + es * m.send_hi, m.count, dt, H->rank + 1, H->comm, stream));
      NK(g_nccl.Recv(f[k] + es * m.recv_hi, m.count, dt, H->rank + 1, H->comm, stream));
    }
  }
  NK(g_nccl.GroupEnd());
  return CSPH_OK;
}

// The same exchange between strips of one process (MULTI): strip r pulls its ghost rows
// and ghost flags from r-1 / r+1 with peer copies on `stream` (its own device current).
static int halo_peer(csph* H, int r, int q, cudaStream_t stream) {
  Strip& s = H->s[r];
  const int n = (int)H->s.size();
  const HaloMap m = halo_map(s, q);
  const size_t es = (size_t)s.v.prec;
  char* f[4];
  state_fields(s.v, q, f);
  if (r > 0) {  // my ghost rows below <- the last owned rows of r-1
    const Strip& o = H->s[r - 1];
    const HaloMap mo = halo_map(o, q);
    char* g[4];
    state_fields(o.v, q, g);
    for (int k = 0; k < 4; ++k)
      CK(cudaMemcpyPeerAsync(f[k] + es * m.recv_lo, s.dev, g[k] + es * mo.send_hi, o.dev,
                             m.count * es, stream));
    CK(cudaMemcpyPeerAsync(s.gflag + m.frecv_lo, s.dev, o.tflag + mo.fsend_hi, o.dev,
                           (size_t)s.ntx, stream));
  }
  if (r < n - 1) {  // my ghost rows above <- the first owned rows of r+1
    const Strip& o = H->s[r + 1];
    const HaloMap mo = halo_map(o, q);
    char* g[4];
    state_fields(o.v, q, g);
    for (int k = 0; k < 4; ++k)
      CK(cudaMemcpyPeerAsync(f[k] + es * m.recv_hi, s.dev, g[k] + es * mo.send_lo, o.dev,
                             m.count * es, stream));
    CK(cudaMemcpyPeerAsync(s.gflag + m.frecv_hi, s.dev, o.tflag + mo.fsend_lo, o.dev,
                           (size_t)s.ntx, stream));
  }
  return CSPH_OK;
}

// Eq.7 maxima and the negative-depth flag over all ranks: max of the u64 bit patterns
// (exact, order-free).
static int allreduce_nccl(csph* H, cudaStream_t stream) {
  Strip& s = H->s[0];
  NK(g_nccl.AllReduce(s.gM, s.gM, 4, ncclUint64, ncclMax, H->comm, stream));
  return CSPH_OK;
}

// MULTI: combine the 4 accumulator slots of every strip on strip 0 and send the result
// back, after each strip's `ready` event; each strip's stream then continues after it.
static int gather_multi(csph* H, cudaEvent_t Strip::*ready) {
  const int n = (int)H->s.size();
  Strip& s0 = H->s[0];
  CK(cudaSetDevice(s0.dev));
  for (int r = 0; r < n; ++r) {
    CK(cudaStreamWaitEvent(s0.st, H->s[r].*ready, 0));
    CK(cudaMemcpyPeerAsync(H->gather + 4 * r, s0.dev, H->s[r].gM, H->s[r].dev,
                           4 * sizeof(unsigned long long), s0.st));
  }
  max_gather_kernel<<<1, 32, 0, s0.st>>>(s0.gM, H->gather, n);
  H->launches += 1;
  CK(cudaGetLastError());
  CK(cudaEventRecord(s0.ev, s0.st));
  for (int r = 1; r < n; ++r) {
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamWaitEvent(s.st, s0.ev, 0));
    CK(cudaMemcpyPeerAsync(s.gM, s.dev, s0.gM, s0.dev, 4 * sizeof(unsigned long long), s.st));
    CK(cudaEventRecord(s.ev, s.st));
  }
  // strip 0's ctrl kernel clears s0.gM: only after every strip has taken its copy
  CK(cudaSetDevice(s0.dev));
  for (int r = 1; r < n; ++r) CK(cudaStreamWaitEvent(s0.st, H->s[r].ev, 0));
  return CSPH_OK;
}

// Halo exchange of buffer q and the maxima combine, all on the strips' main streams
// (staged path and set_state).  NCCL for DIST, peer copies for MULTI.
static int exchange(csph* H, int q) {
  if (H->mode == DIST) {
    int st = halo_nccl(H, q, H->s[0].st);
    if (st) return st;
    return allreduce_nccl(H, H->s[0].st);
  }
  if (H->mode == MULTI) {
    const int n = (int)H->s.size();
    for (int r = 0; r < n; ++r) {
      CK(cudaSetDevice(H->s[r].dev));
      CK(cudaEventRecord(H->s[r].ev, H->s[r].st));
    }
    int st = gather_multi(H, &Strip::ev);
    if (st) return st;
    // every strip's state of buffer q is final (gather waited for all): pull the halos
    for (int r = 0; r < n; ++r) {
      Strip& s = H->s[r];
      CK(cudaSetDevice(s.dev));
      if (r == 0) CK(cudaStreamWaitEvent(s.st, H->s[0].ev, 0));
      if ((st = halo_peer(H, r, q, s.st))) return st;
    }
    // every strip must finish reading its neighbours before they run ahead
    for (int r = 0; r < n; ++r) {
      CK(cudaSetDevice(H->s[r].dev));
      CK(cudaEventRecord(H->s[r].ev, H->s[r].st));
    }
    for (int r = 0; r < n; ++r) {
      CK(cudaSetDevice(H->s[r].dev));
      if (r > 0) CK(cudaStreamWaitEvent(H->s[r].st, H->s[r - 1].ev, 0));
      if (r < n - 1) CK(cudaStreamWaitEvent(H->s[r].st, H->s[r + 1].ev, 0));
    }
  }
  return CSPH_OK;
}

// Input validation on the device (CSPH_EINVAL on NaN/Inf, h < 0, psi
// outside [0,1)); bit 3 = psi is not uniform over this strip's rows.
__global__ void validate_kernel(StripView S, int jlo, int jhi, const double* psi, double psi0,
                                int* flags, int buf) {
  // grid-stride over rows, flags accumulated per thread, one atomicOr per block (a per-warp
  // atomic on one word serialises: with a psi field every warp sets bit 3)
  __shared__ int bf;
  if (threadIdx.x == 0 && threadIdx.y == 0) bf = 0;
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < S.nx) {
    for (int j = jlo + (int)(blockIdx.y * blockDim.y + threadIdx.y); j < jhi;
         j += (int)(gridDim.y * blockDim.y)) {
      const size_t c = off(S.pitch, i, j);
      const double H = S.H[buf][c], qx = S.Qx[buf][c], qy = S.Qy[buf][c], b = S.b[buf][c];
      if (!isfinite(H) || !isfinite(qx) || !isfinite(qy) || !isfinite(b)) f |= 1;
      if (H < 0.0) f |= 2;
      if (psi) {
        const double p = psi[c];
        if (!(p >= 0.0 && p < 1.0)) f |= 4;
        if (p != psi0) f |= 8;
      }
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(&bf, f);
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0 && bf) atomicOr(flags, bf);
}

static double* src_dst0(const StripView& v, int k) {
  return k == 0 ? v.H[0] : k == 1 ? v.Qx[0] : k == 2 ? v.Qy[0] : v.b[0];
}

static int upload_rows(csph* H, Strip& s, int j_begin, int j_end, const double* h,
                       const double* hu, const double* hv, const double* b, const double* psi) {
  // rows of this strip incl. halo rows where a neighbour exists
  StripView& v = s.v;
  int lo = s.gj0 - (v.wall_lo ? 0 : GY);
  int hi = s.gj0 + v.ny + (v.wall_hi ? 0 : GY);
  if (lo < j_begin || hi > j_end)
    return fail(CSPH_EINVAL, "rows [%d,%d) do not cover strip rows [%d,%d) + halo", j_begin,
                j_end, lo, hi);
  const int nx = H->nx;
  const int ub = v.prec == 4 ? 1 : 0;  // fp32 mode: fp64 upload into buffer 1, then convert
  const double* src[4] = {h, hu, hv, b};
  double* dst[4] = {v.H[ub], v.Qx[ub], v.Qy[ub], v.b[ub]};
  for (int k = 0; k < 4; ++k) {
    const double* a = src[k] + (size_t)(lo - j_begin) * nx;
    double* d = dst[k] + off(v.pitch, 0, lo - s.gj0);
    CK(cudaMemcpy2DAsync(d, (size_t)v.pitch * 8, a, (size_t)nx * 8, (size_t)nx * 8, hi - lo,
                         cudaMemcpyHostToDevice, s.st));
  }
  double* psid = nullptr;
  double psi0 = 0.0;
  if (psi) {
    size_t n = (size_t)(v.ny + 2 * GY) * v.pitch;
    if (!s.Wbuf) {
      int st = dalloc(s, (void**)&s.Wbuf, n * 8);
      if (st) return st;
      CK(cudaMemsetAsync(s.Wbuf, 0, n * 8, s.st));
    }
    psid = s.Wbuf;
    psi0 = psi[(size_t)(lo - j_begin) * nx];
    CK(cudaMemcpy2DAsync(psid + off(v.pitch, 0, lo - s.gj0), (size_t)v.pitch * 8,
                         psi + (size_t)(lo - j_begin) * nx, (size_t)nx * 8, (size_t)nx * 8,
                         hi - lo, cudaMemcpyHostToDevice, s.st));
  }
  CK(cudaMemsetAsync(s.dflags, 0, sizeof(int), s.st));
  {
    const int bx = (nx + 31) / 32;
    const int by = std::max(1, std::min((hi - lo + 7) / 8, (8 * 148 + bx - 1) / bx));
    dim3 blk(32, 8), grd(bx, by);
    validate_kernel<<<grd, blk, 0, s.st>>>(v, lo - s.gj0, hi - s.gj0, psid, psi0, s.dflags, ub);
    CK(cudaGetLastError());
  }
  int flags = 0;
  CK(cudaMemcpyAsync(&flags, s.dflags, sizeof(int), cudaMemcpyDeviceToHost, s.st));
  CK(cudaStreamSynchronize(s.st));
  if (flags & 1) return fail(CSPH_EINVAL, "non-finite input value");
  if (flags & 2) return fail(CSPH_EINVAL, "negative depth in input");
  if (flags & 4) return fail(CSPH_EINVAL, "psi outside [0,1)");
  const size_t ntot = (size_t)(v.ny + 2 * GY) * v.pitch;
  if (v.prec == 4) {
    for (int k = 0; k < 4; ++k)
      to_f32_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, s.st>>>((float*)src_dst0(v, k),
                                                                      dst[k], ntot);
    CK(cudaGetLastError());
  }
  if (!psi || !(flags & 8)) {
    // uniform porosity: W is a scalar (64 B/cell instead of 72 B/cell)
    v.W = nullptr;
    v.Wc = 1.0 / (1.0 - psi0);
  } else {
    w_from_psi_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, s.st>>>(s.Wbuf, s.Wbuf, ntot);
    CK(cudaGetLastError());
    v.W = s.Wbuf;
    if (v.prec == 4) {
      if (!s.Wbuf32) {
        int st = dalloc(s, (void**)&s.Wbuf32, ntot * 4);
        if (st) return st;
      }
      to_f32_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, s.st>>>(s.Wbuf32, s.Wbuf, ntot);
      CK(cudaGetLastError());
      v.W = (const double*)s.Wbuf32;  // holds fp32 values
    }
  }
  return CSPH_OK;
}

// Tile rows from the state: with HGS only tiles holding water do real work,
// so the tiling must give enough of them to fill the GPU -- the largest ty in 128..16 whose
// wet tiles make 2.5 waves of 3 resident CTAs per SM -- while keeping the launch of the
// skipped ones cheap (at most 40 K tiles in all).  Measured on one B200: C3 4096^2 -> 32 rows
// (+22 % over 128), C4 8192^2 -> 64 (+9 %), C5 16384^2 -> 128.
static int order_reset(csph* H, Strip& s);

static int choose_tile_rows(csph* H, Strip& s, int buf = 0) {
  const int nby = (s.v.ny + kTyMin - 1) / kTyMin;
  dim3 grd((unsigned)s.ntx, (unsigned)nby);
  if (s.v.prec == 4)
    wet_blocks_kernel<float><<<grd, FUSED_NT, 0, s.st>>>(s.v, H->P.eps, s.wetblk, buf);
  else
    wet_blocks_kernel<double><<<grd, FUSED_NT, 0, s.st>>>(s.v, H->P.eps, s.wetblk, buf);
  H->launches += 1;
  CK(cudaGetLastError());
  std::vector<unsigned char> w((size_t)s.ntx * nby);
  CK(cudaMemcpyAsync(w.data(), s.wetblk, w.size(), cudaMemcpyDeviceToHost, s.st));
  CK(cudaStreamSynchronize(s.st));
  const long long want = 5LL * FUSED_MINB * s.nsm / 2;
  int pick = 0;
  static const int kTys[] = {192, 128, 64, 32, 16};  // with the costliest-first order (7.5)
  for (int ty : kTys) {
    const int f = ty / kTyMin, nty = (s.v.ny + ty - 1) / ty;
    if ((long long)nty * s.ntx > 40000) break;  // finer tilings only add skipped-CTA overhead
    long long wet = 0;
    for (int r = 0; r < nty; ++r)
      for (int q = 0; q < s.ntx; ++q) {
        bool any = false;
        for (int k = r * f; k < (r + 1) * f && k < nby && !any; ++k) any = w[(size_t)k * s.ntx + q];
        wet += any;
      }
    pick = ty;
    if (wet >= want) break;
  }
  s.ty = pick ? pick : 128;
  s.nty = (s.v.ny + s.ty - 1) / s.ty;
  return CSPH_OK;
}

int csph_set_state_rows(csph_t* H, int j_begin, int j_end, const double* h, const double* hu,
                        const double* hv, const double* b, const double* psi) {
  if (!H || !h || !hu || !hv || !b) return fail(CSPH_EINVAL, "NULL argument");
  if (j_begin < 0 || j_end > H->ny || j_end <= j_begin) return fail(CSPH_EINVAL, "bad row range");
  H->have_state = false;
  graphs_reset(H);
  int st;
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    if ((st = upload_rows(H, s, j_begin, j_end, h, hu, hv, b, psi))) return st;
    if (s.auto_ty && H->p.path == CSPH_PATH_FUSED && (st = choose_tile_rows(H, s))) return st;
    if ((st = order_reset(H, s))) return st;
    init_ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl);
    CK(cudaMemsetAsync(s.gM, 0, 4 * sizeof(unsigned long long), s.st));
    CK(cudaMemsetAsync(s.tflag, HGS_ALL, 2 * s.tflag_cap, s.st));  // all tiles active
    CK(cudaMemsetAsync(s.tstate, 0, s.tflag_cap, s.st));
    CK(cudaMemsetAsync(s.gflag, HGS_ALL, 4 * (size_t)s.ntx, s.st));
    CK(cudaMemsetAsync(s.hstats, 0, 4 * sizeof(unsigned long long), s.st));
    // walls: ghosts of buffer 0 (W is read only on owned cells: no ghosts needed)
    launch_mirror(s.v, s.ctrl, 0, s.st, &H->launches);
    CK(cudaGetLastError());
  }
  // a new run restarts the combine's sequence numbers: clear the inboxes (before the
  // initial combine below, which no rank passes before every rank got here)
  for (auto& s : H->s)
    if (s.inbox) {
      CK(cudaSetDevice(s.dev));
      CK(cudaMemsetAsync(s.inbox, 0, 2 * (size_t)H->nranks * kInboxW * sizeof(unsigned long long),
                         s.st));
    }
  // maxima of the initial state, combined across strips / ranks
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    dim3 blk(32, 8), grd((s.v.nx + 31) / 32, (s.v.ny + 7) / 8);
    if (s.v.prec == 4)
      maxima32_kernel<<<grd, blk, 0, s.st>>>(s.v, s.ctrl, H->P, s.gM);
    else
      maxima_kernel<<<grd, blk, 0, s.st>>>(s.v, s.ctrl, H->P, s.gM);
    CK(cudaGetLastError());
  }
  if (H->mode == DIST) {
    Strip& s = H->s[0];
    NK(g_nccl.AllReduce(s.gM, s.gM, 4, ncclUint64, ncclMax, H->comm, s.st));
  } else if (H->mode == MULTI) {
    if ((st = exchange(H, 0))) return st;  // also refreshes halos of buffer 0
  }
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl, s.gM, s.Mlast, s.dtlog, s.limlog, H->P, 0);
    CK(cudaGetLastError());
  }
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.st));
  }
  H->have_state = true;
  H->host_parity = 0;
  return CSPH_OK;
}

static int upload_field_rows(Strip& s, double* dst, const double* src_rows, int j_begin,
                             int lo, int hi, int nx) {
  const StripView& v = s.v;
  CK(cudaMemcpy2DAsync(dst + off(v.pitch, 0, lo - s.gj0), (size_t)v.pitch * 8,
                       src_rows + (size_t)(lo - j_begin) * nx, (size_t)nx * 8, (size_t)nx * 8,
                       hi - lo, cudaMemcpyHostToDevice, s.st));
  return CSPH_OK;
}

int csph_set_fields_rows(csph_t* H, int j_begin, int j_end, const double* n_manning,
                         const double* beta, const double* src) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  graphs_reset(H);
  if (j_begin < 0 || j_end > H->ny || j_end <= j_begin) return fail(CSPH_EINVAL, "bad row range");
  if (H->p.precision == 32)
    return fail(CSPH_EINVAL, "csph_set_fields: the fp32 mode runs the hot-path features only");
  const bool has_n = n_manning != nullptr, has_src = beta != nullptr || src != nullptr;
  const int nx = H->nx;
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    StripView& v = s.v;
    const int lo = s.gj0 - (v.wall_lo ? 0 : GY);
    const int hi = s.gj0 + v.ny + (v.wall_hi ? 0 : GY);
    if (lo < j_begin || hi > j_end)
      return fail(CSPH_EINVAL, "rows [%d,%d) do not cover strip rows [%d,%d) + halo", j_begin,
                  j_end, lo, hi);
    const size_t n = (size_t)(v.ny + 2 * GY) * v.pitch;
    int st;
    double *cg = nullptr, *bt = nullptr, *sr = nullptr, *aj = nullptr;
    if (has_n) {
      if (!s.cgbuf && (st = dalloc(s, (void**)&s.cgbuf, n * 8))) return st;
      cg = s.cgbuf;
      if (H->p.aj_mode == 1) {
        if (!s.ajbuf && (st = dalloc(s, (void**)&s.ajbuf, n * 8))) return st;
        aj = s.ajbuf;
        CK(cudaMemsetAsync(aj, 0, n * 8, s.st));
      }
      CK(cudaMemsetAsync(cg, 0, n * 8, s.st));
      if ((st = upload_field_rows(s, cg, n_manning, j_begin, lo, hi, nx))) return st;
    }
    if (has_src) {
      if (!s.betabuf && (st = dalloc(s, (void**)&s.betabuf, n * 8))) return st;
      if (!s.srcbuf && (st = dalloc(s, (void**)&s.srcbuf, n * 8))) return st;
      bt = s.betabuf;
      sr = s.srcbuf;
      CK(cudaMemsetAsync(bt, 0, n * 8, s.st));
      CK(cudaMemsetAsync(sr, 0, n * 8, s.st));
      if (beta && (st = upload_field_rows(s, bt, beta, j_begin, lo, hi, nx))) return st;
      if (src && (st = upload_field_rows(s, sr, src, j_begin, lo, hi, nx))) return st;
    }
    CK(cudaMemsetAsync(s.dflags, 0, sizeof(int), s.st));
    dim3 blk(32, 8), grd((nx + 31) / 32, (hi - lo + 7) / 8);
    fields_kernel<<<grd, blk, 0, s.st>>>(v, cg, bt, sr, aj, lo - s.gj0, hi - s.gj0, H->p.g,
                                         H->p.n_manning, has_n, beta != nullptr,
                                         src != nullptr, s.dflags);
    CK(cudaGetLastError());
    int flags = 0;
    CK(cudaMemcpyAsync(&flags, s.dflags, sizeof(int), cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    if (flags & 1) return fail(CSPH_EINVAL, "n_manning field must be finite and >= 0");
    if (flags & 2) return fail(CSPH_EINVAL, "beta field must be finite and >= 0");
    if (flags & 4) return fail(CSPH_EINVAL, "source field must be finite and >= 0");
    for (double* F : {cg, bt, sr, aj}) {
      if (!F) continue;
      int n1 = (v.ny + 2 * GY) * 6, n2 = (v.nx + 6) * 6;
      mirror_field_kernel<<<(n1 + 255) / 256, 256, 0, s.st>>>(v, F);
      mirror_field_y_kernel<<<(n2 + 255) / 256, 256, 0, s.st>>>(v, F);
    }
    CK(cudaGetLastError());
    v.cg = cg;
    v.beta = bt;
    v.src = sr;
    v.aj0 = aj;
    // new source fields change which dry tiles are identities: every tile marches again
    // (tstate >= 2 would skip tiles whose two buffers differ once sources stop)
    CK(cudaMemsetAsync(s.tflag, HGS_ALL, 2 * s.tflag_cap, s.st));
    CK(cudaMemsetAsync(s.tstate, 0, s.tflag_cap, s.st));
    CK(cudaMemsetAsync(s.gflag, HGS_ALL, 4 * (size_t)s.ntx, s.st));
  }
  H->P.fric = H->p.n_manning > 0.0 || has_n;
  return CSPH_OK;
}

int csph_set_fields(csph_t* H, const double* n_manning, const double* beta, const double* src) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  return csph_set_fields_rows(H, 0, H->ny, n_manning, beta, src);
}

int csph_set_state(csph_t* H, const double* h, const double* hu, const double* hv,
                   const double* b, const double* psi) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  return csph_set_state_rows(H, 0, H->ny, h, hu, hv, b, psi);
}

static Hgs hgs_of(const csph* H, const Strip& s) {
  Hgs h;
  const size_t nt = (size_t)s.ntx * s.nty;
  h.fprev = s.tflag + nt * (size_t)H->host_parity;
  h.fnext = s.tflag + nt * (size_t)(H->host_parity ^ 1);
  h.tstate = s.tstate;
  // ghost flags of parity host_parity, written by the previous step's exchange
  const unsigned char* g = s.gflag + 2 * (size_t)s.ntx * (size_t)H->host_parity;
  h.glo = s.v.wall_lo ? nullptr : g;
  h.ghi = s.v.wall_hi ? nullptr : g + s.ntx;
  h.ntx = s.ntx;
  h.nty = s.nty;
  h.enable = H->p.hgs != 0 && H->p.path == CSPH_PATH_FUSED;
  h.stats = s.hstats;
  h.order = nullptr;
  h.cost = s.tcost + s.tflag_cap * (size_t)H->host_parity;
  return h;
}

// The launch order of this step's ordered launch, tile rows [tr0, tr1):
// join the sort made during the previous step, then fork the next step's sort onto the
// order stream (from the costs of the step before this one), beside this step's kernel.
static int order_step(csph* H, Strip& s, int tr0, int tr1, Hgs& hg) {
  if (!hg.enable || tr1 <= tr0) return CSPH_OK;
  const int p = H->host_parity;
  const size_t cap = s.tflag_cap;
  if (s.osort_pending) {
    CK(cudaStreamWaitEvent(s.st, s.ev_ojoin, 0));
    s.osort_pending = false;
  }
  hg.order = s.torder + cap * (size_t)p;
  CK(cudaEventRecord(s.ev_ofork, s.st));
  CK(cudaStreamWaitEvent(s.ost, s.ev_ofork, 0));
  launch_order_tiles(s.tcost + cap * (size_t)(p ^ 1), s.ntx, tr0, tr1,
                     s.torder + cap * (size_t)(p ^ 1), s.ost, &H->launches);
  CK(cudaGetLastError());
  CK(cudaEventRecord(s.ev_ojoin, s.ost));
  s.osort_pending = true;
  return CSPH_OK;
}

// The main stream waits for a pending sort (before a capture ends or starts, at the end of
// csph_step, before the order buffers are reset).
static int order_join(Strip& s) {
  if (s.osort_pending) {
    CK(cudaStreamWaitEvent(s.st, s.ev_ojoin, 0));
    s.osort_pending = false;
  }
  return CSPH_OK;
}

// Natural order and zero costs for both parities (a new state or tiling).
static int order_reset(csph* H, Strip& s) {
  int st;
  if ((st = order_join(s))) return st;
  CK(cudaMemsetAsync(s.tcost, 0, 2 * s.tflag_cap * sizeof(unsigned short), s.st));
  launch_order_identity(s.torder, (int)(2 * s.tflag_cap), s.st, &H->launches);
  CK(cudaGetLastError());
  return CSPH_OK;
}

// One step of a single-grid handle: the 3 launches (clear flags, step kernel(s), ctrl)
// reading buffer host_parity.  Used directly and inside the CUDA-graph capture.
static int single_step(csph* H, Strip& s) {
  if (H->p.path == CSPH_PATH_STAGED) {
    launch_staged_step(s.v, s.ctrl, s.scr, H->P, s.gM, s.st, &H->launches);
    launch_mirror(s.v, s.ctrl, 1, s.st, &H->launches);
  } else {
    Hgs hg = hgs_of(H, s);
    int st;
    if ((st = order_step(H, s, 0, s.nty, hg))) return st;  // costliest tiles first
    launch_fused_step(s.v, s.ctrl, H->P, s.gM, 0, s.v.ny, s.ty, hg, s.st, &H->launches);
  }
  CK(cudaGetLastError());
  ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl, s.gM, s.Mlast, s.dtlog, s.limlog, H->P, 1);
  H->launches += 1;
  CK(cudaGetLastError());
  H->host_parity ^= 1;
  return CSPH_OK;
}

static int split_step(csph* H, int n, int q);

// One step of a graph-replayed handle: the single-grid launches, or (DIST) the split
// launches with the NCCL halo and allreduce on the comm stream (captured into the same graph:
// the comm stream joins the capture through ev_edge and rejoins it through ev_comm).
static int capture_step(csph* H, Strip& s) {
  if (H->mode != DIST) return single_step(H, s);
  const int q = H->host_parity ^ 1;
  const int st = split_step(H, 0, q);
  H->host_parity = q;
  return st;
}

// Two steps from buffer parity p as one CUDA graph (captured once, replayed).
static int graph_pair(csph* H, Strip& s, long long* per_launch) {
  cudaGraphExec_t& ge = H->gexec[H->host_parity];
  if (!ge) {
    const long long l0 = H->launches;
    const int p0 = H->host_parity;
    cudaGraph_t gr = nullptr;
    // capture on a private stream (the legacy default stream cannot be captured); the
    // graph is then launched on the handle's stream
    if (!H->cap) CK(cudaStreamCreateWithFlags(&H->cap, cudaStreamNonBlocking));
    const cudaStream_t user = s.st;
    int st;
    if ((st = order_join(s))) return st;  // no dependency on work outside the capture
    s.st = H->cap;
    cudaError_t e = cudaStreamBeginCapture(s.st, cudaStreamCaptureModeRelaxed);
    st = e == cudaSuccess ? CSPH_OK : fail(CSPH_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    if (!st) st = capture_step(H, s);
    if (!st) st = capture_step(H, s);
    if (!st) st = order_join(s);  // every forked sort rejoins the capture
    e = cudaStreamEndCapture(s.st, &gr);
    s.st = user;
    H->host_parity = p0;
    if (st) return st;
    if (e != cudaSuccess) return fail(CSPH_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    const cudaError_t e2 = cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphDestroy(gr);
    if (e2 != cudaSuccess) {
      ge = nullptr;
      return fail(CSPH_ECUDA, "graph instantiate: %s", cudaGetErrorString(e2));
    }
    H->graph_kernels = H->launches - l0;
    H->launches = l0;
  }
  CK(cudaGraphLaunch(ge, s.st));
  *per_launch = H->graph_kernels;
  return CSPH_OK;
}

// The boundary tile rows of a strip, [0, lo) and [hi, ny), hold the GY rows each
// neighbour needs; the halo exchange starts after them and overlaps the interior
// [lo, hi).  Both are whole tile rows (the HGS tiling), and the last one must hold at
// least GY rows: a short last tile (ny % ty in {1, 2}) is merged with the one before it,
// else rows the neighbour receives would still be in flight in the interior launch.
// false: no interior tile row, the strip is launched whole before the exchange.
static bool edge_split(const Strip& s, int* lo, int* hi) {
  const int ny = s.v.ny, ty = s.ty;
  int l = ty, h = (s.nty - 1) * ty;
  if (ny - h < GY) h -= ty;
  if (s.nty < 3 || h <= l) return false;
  *lo = l;
  *hi = h;
  return true;
}

// One step of a DIST or MULTI handle on the fused path: edge tile rows, then the halo
// exchange of buffer q on the comm streams (NCCL send/recv or peer copies) overlapped
// with the interior, then the combine of the Eq.7 maxima and the negative-depth flag, and
// the ctrl kernel once the halo has landed.
static int push_step(csph* H, int n);

static int split_step(csph* H, int n, int q) {
  if (H->push) return push_step(H, n);
  const int ns = (int)H->s.size();
  std::vector<int> lo(ns, 0), hi(ns, 0);
  std::vector<char> sp(ns, 0);
  for (int r = 0; r < ns; ++r) {  // 1. edge tile rows
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    const Hgs hg = hgs_of(H, s);
    if (H->profiling && r == 0) CK(cudaEventRecord(H->evs[2 * n], s.st));
    sp[r] = edge_split(s, &lo[r], &hi[r]);
    if (sp[r]) {
      launch_fused_step(s.v, s.ctrl, H->P, s.gM, 0, lo[r], s.ty, hg, s.st, &H->launches);
      launch_fused_step(s.v, s.ctrl, H->P, s.gM, hi[r], s.v.ny, s.ty, hg, s.st, &H->launches);
    } else {
      launch_fused_step(s.v, s.ctrl, H->P, s.gM, 0, s.v.ny, s.ty, hg, s.st, &H->launches);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(s.ev_edge, s.st));
  }
  int st;
  for (int r = 0; r < ns; ++r) {  // 2. halo exchange on the comm streams
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamWaitEvent(s.cst, s.ev_edge, 0));
    if (H->mode == DIST) {
      if ((st = halo_nccl(H, q, s.cst))) return st;
    } else {
      if (r > 0) CK(cudaStreamWaitEvent(s.cst, H->s[r - 1].ev_edge, 0));
      if (r < ns - 1) CK(cudaStreamWaitEvent(s.cst, H->s[r + 1].ev_edge, 0));
      if ((st = halo_peer(H, r, q, s.cst))) return st;
      CK(cudaEventRecord(s.ev_comm, s.cst));
    }
  }
  for (int r = 0; r < ns; ++r) {  // 3. interior tile rows
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    if (sp[r]) {
      Hgs hg = hgs_of(H, s);
      // the interior tile rows, costliest first
      if ((st = order_step(H, s, lo[r] / s.ty, hi[r] / s.ty, hg))) return st;
      launch_fused_step(s.v, s.ctrl, H->P, s.gM, lo[r], hi[r], s.ty, hg, s.st, &H->launches);
    }
    if (H->profiling && r == 0) CK(cudaEventRecord(H->evs[2 * n + 1], s.st));
    CK(cudaGetLastError());
    CK(cudaEventRecord(s.ev_int, s.st));
  }
  if (H->mode == DIST) {  // 4. combine, then ctrl after the halo and the allreduce
    Strip& s = H->s[0];
    CK(cudaStreamWaitEvent(s.cst, s.ev_int, 0));
    if ((st = allreduce_nccl(H, s.cst))) return st;
    CK(cudaEventRecord(s.ev_comm, s.cst));
    CK(cudaStreamWaitEvent(s.st, s.ev_comm, 0));
  } else {
    if ((st = gather_multi(H, &Strip::ev_int))) return st;
    // ctrl (and the next step) after my halo landed and my neighbours finished reading
    // my edge rows of buffer q (the step after next overwrites them)
    for (int r = 0; r < ns; ++r) {
      Strip& s = H->s[r];
      CK(cudaSetDevice(s.dev));
      for (int o = r - 1; o <= r + 1; ++o)
        if (o >= 0 && o < ns) CK(cudaStreamWaitEvent(s.st, H->s[o].ev_comm, 0));
    }
  }
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl, s.gM, s.Mlast, s.dtlog, s.limlog, H->P, 1);
    H->launches += 1;
    CK(cudaGetLastError());
  }
  return CSPH_OK;
}

// One step of a DIST or MULTI handle whose strips push their halos: every strip
// launched whole (its edge tile rows write the neighbours' ghost rows and flags from inside
// the kernel), then the combine of the Eq.7 maxima and the negative-depth flag -- which is
// also the step's barrier: no strip's next step starts before every strip's kernel (and so
// every push into its ghost rows) is done -- and the ctrl kernels.
static int push_step(csph* H, int n) {
  const int ns = (int)H->s.size();
  int st;
  for (int r = 0; r < ns; ++r) {
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    Hgs hg = hgs_of(H, s);
    if ((st = order_step(H, s, 0, s.nty, hg))) return st;  // costliest tiles first
    if (H->profiling && r == 0) CK(cudaEventRecord(H->evs[2 * n], s.st));
    launch_fused_step(s.v, s.ctrl, H->P, s.gM, 0, s.v.ny, s.ty, hg, s.st, &H->launches);
    if (H->profiling && r == 0) CK(cudaEventRecord(H->evs[2 * n + 1], s.st));
    CK(cudaGetLastError());
    CK(cudaEventRecord(s.ev_int, s.st));
  }
  if (H->p2p_combine) {
    // each ctrl kernel publishes its maxima to every rank's inbox and waits for all
  } else if (H->mode == DIST) {
    Strip& s = H->s[0];
    CK(cudaStreamWaitEvent(s.cst, s.ev_int, 0));
    if ((st = allreduce_nccl(H, s.cst))) return st;
    CK(cudaEventRecord(s.ev_comm, s.cst));
    CK(cudaStreamWaitEvent(s.st, s.ev_comm, 0));
  } else if ((st = gather_multi(H, &Strip::ev_int))) {
    return st;
  }
  for (int r = 0; r < ns; ++r) {
    Strip& s = H->s[r];
    CK(cudaSetDevice(s.dev));
    ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl, s.gM, s.Mlast, s.dtlog, s.limlog, H->P, 1,
                                   combine_of(H, s, H->mode == DIST ? H->rank : r));
    H->launches += 1;
    CK(cudaGetLastError());
  }
  return CSPH_OK;
}

int csph_step(csph_t* H, int nsteps) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (nsteps < 0) return fail(CSPH_EINVAL, "nsteps < 0");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "csph_step before csph_set_state");
  H->launches = 0;
  if (H->profiling && H->evs.size() < (size_t)nsteps * 2) {
    CK(cudaSetDevice(H->s[0].dev));
    while (H->evs.size() < (size_t)nsteps * 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      H->evs.push_back(e);
    }
  }
  // DIST and MULTI (fused path): boundary tile rows first, their halo exchange overlapped
  // with the interior (a single rank takes the same path; its NCCL calls are no-ops)
  const bool split = H->mode != SINGLE && H->p.path == CSPH_PATH_FUSED;
  for (int n = 0; n < nsteps; ++n) {
    const int q = H->host_parity ^ 1;
    if (split) {
      if (H->mode == DIST && H->graphs && !H->profiling && n + 2 <= nsteps) {
        // DIST steps replayed in pairs from CUDA graphs, NCCL calls included
        Strip& s = H->s[0];
        CK(cudaSetDevice(s.dev));
        long long k = 0;
        int st = graph_pair(H, s, &k);
        if (st) return st;
        H->launches += k;
        ++n;
        continue;
      }
      int st = split_step(H, n, q);
      if (st) return st;
      H->host_parity = q;
      continue;
    }
    if (H->mode == SINGLE && H->s.size() == 1 && !H->profiling) {
      // (profiling runs take the strip loop below: events around the step kernel)
      Strip& s = H->s[0];
      CK(cudaSetDevice(s.dev));
      if (H->graphs && n + 2 <= nsteps) {
        long long k = 0;
        int st = graph_pair(H, s, &k);
        if (st) return st;
        H->launches += k;
        ++n;  // two steps replayed; host_parity is back where it was
        continue;
      }
      int st = single_step(H, s);
      if (st) return st;
      continue;
    }
    for (size_t si = 0; si < H->s.size(); ++si) {
      Strip& s = H->s[si];
      CK(cudaSetDevice(s.dev));
      Hgs hg = hgs_of(H, s);
      if (H->p.path != CSPH_PATH_STAGED) {  // costliest tiles first
        int st;
        if ((st = order_step(H, s, 0, s.nty, hg))) return st;
      }
      if (H->profiling && si == 0) CK(cudaEventRecord(H->evs[2 * n], s.st));
      if (H->p.path == CSPH_PATH_STAGED)
        launch_staged_step(s.v, s.ctrl, s.scr, H->P, s.gM, s.st, &H->launches);
      else
        launch_fused_step(s.v, s.ctrl, H->P, s.gM, 0, s.v.ny, s.ty, hg, s.st,
                          &H->launches);  // writes the wall ghosts in its epilogue
      if (H->profiling && si == 0) CK(cudaEventRecord(H->evs[2 * n + 1], s.st));
      if (H->p.path == CSPH_PATH_STAGED) launch_mirror(s.v, s.ctrl, 1, s.st, &H->launches);
      CK(cudaGetLastError());
    }
    int st = exchange(H, q);
    if (st) return st;
    for (auto& s : H->s) {
      CK(cudaSetDevice(s.dev));
      ctrl_kernel<<<1, 1, 0, s.st>>>(s.ctrl, s.gM, s.Mlast, s.dtlog, s.limlog, H->P, 1);
      H->launches += 1;
      CK(cudaGetLastError());
    }
    H->host_parity = q;
  }
  int status = 0;
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    if ((status = order_join(s))) return status;
  }
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    Ctrl c;
    CK(cudaMemcpyAsync(&c, s.ctrl, sizeof c, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    if (c.status && !status) status = c.status;
  }
  if (H->profiling) {
    CK(cudaSetDevice(H->s[0].dev));
    for (int n = 0; n < nsteps; ++n) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, H->evs[2 * n], H->evs[2 * n + 1]));
      H->prof_ms += ms;
    }
    H->prof_steps += nsteps;
  }
  if (status) return fail(status, "%s", csph_strerror(status));
  return CSPH_OK;
}

static int read_ctrl(csph* H, Ctrl* c) {
  Strip& s = H->s[0];
  CK(cudaSetDevice(s.dev));
  CK(cudaMemcpyAsync(c, s.ctrl, sizeof *c, cudaMemcpyDeviceToHost, s.st));
  CK(cudaStreamSynchronize(s.st));
  return CSPH_OK;
}

int csph_get_state_rows(csph_t* H, int j_begin, int j_end, double* h, double* hu, double* hv,
                        double* b) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "no state");
  if (j_begin < 0 || j_end > H->ny || j_end <= j_begin) return fail(CSPH_EINVAL, "bad row range");
  for (auto& s : H->s) {
    Ctrl c;
    CK(cudaSetDevice(s.dev));
    CK(cudaMemcpyAsync(&c, s.ctrl, sizeof c, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    const StripView& v = s.v;
    int lo = s.gj0 > j_begin ? s.gj0 : j_begin;
    int hi = s.gj0 + v.ny < j_end ? s.gj0 + v.ny : j_end;
    if (hi <= lo) continue;
    const int p = c.parity;
    double* dst[4] = {h, hu, hv, b};
    const double* src[4] = {v.H[p], v.Qx[p], v.Qy[p], v.b[p]};
    const size_t ntot = (size_t)(v.ny + 2 * GY) * v.pitch;
    if (v.prec == 4 && !s.tmpd) {
      int st = dalloc(s, (void**)&s.tmpd, ntot * 8);
      if (st) return st;
    }
    for (int k = 0; k < 4; ++k) {
      if (!dst[k]) continue;
      const double* sk = src[k];
      if (v.prec == 4) {  // widen the fp32 field first
        to_f64_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, s.st>>>(s.tmpd, (const float*)sk,
                                                                         ntot);
        CK(cudaGetLastError());
        sk = s.tmpd;
      }
      CK(cudaMemcpy2DAsync(dst[k] + (size_t)(lo - j_begin) * H->nx, (size_t)H->nx * 8,
                           sk + off(v.pitch, 0, lo - s.gj0), (size_t)v.pitch * 8,
                           (size_t)H->nx * 8, hi - lo, cudaMemcpyDeviceToHost, s.st));
    }
    CK(cudaStreamSynchronize(s.st));
  }
  return CSPH_OK;
}

int csph_get_state(csph_t* H, double* h, double* hu, double* hv, double* b) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  return csph_get_state_rows(H, 0, H->ny, h, hu, hv, b);
}

// Asynchronous Save (the Save block records states every 100-1000 iterations,
// CUDA streams separating the CPU<->GPU copies from the computation).  On the step stream:
// wait until the previous Save has left the snapshot, then copy the owned rows of the state
// (widened to fp64 in fp32 mode) into the dense snapshot; on the save stream: wait for that
// copy, then move the snapshot to the caller's arrays.  Later csph_step calls run on the step
// stream while the device->host copy drains, and never touch the snapshot.
int csph_save_begin(csph_t* H, double* h, double* hu, double* hv, double* b) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "no state");
  double* dst[4] = {h, hu, hv, b};
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    const StripView& v = s.v;
    const size_t plane = (size_t)v.ny * H->nx;
    if (!s.sst) {
      CK(cudaStreamCreateWithFlags(&s.sst, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&s.ev_snap, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s.ev_saved, cudaEventDisableTiming));
    }
    if (!s.snap) {
      int st = dalloc(s, (void**)&s.snap, 4 * plane * 8);
      if (st) return st;
    }
    const size_t ntot = (size_t)(v.ny + 2 * GY) * v.pitch;
    if (v.prec == 4 && !s.tmpd) {
      int st = dalloc(s, (void**)&s.tmpd, ntot * 8);
      if (st) return st;
    }
    // the buffer holding the state: the ctrl block's parity once the launched steps are done
    // (a frozen step, CSPH_ENEGDEPTH, does not flip it); the steps are complete on return
    // from csph_step, so this read does not wait for device work
    Ctrl c;
    CK(cudaMemcpyAsync(&c, s.ctrl, sizeof c, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    const int p = c.parity;
    const double* src[4] = {v.H[p], v.Qx[p], v.Qy[p], v.b[p]};
    if (s.save_issued) CK(cudaStreamWaitEvent(s.st, s.ev_saved, 0));
    for (int k = 0; k < 4; ++k) {
      if (!dst[k]) continue;
      const double* sk = src[k];
      if (v.prec == 4) {
        to_f64_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, s.st>>>(s.tmpd, (const float*)sk,
                                                                         ntot);
        CK(cudaGetLastError());
        sk = s.tmpd;
      }
      CK(cudaMemcpy2DAsync(s.snap + k * plane, (size_t)H->nx * 8, sk + off(v.pitch, 0, 0),
                           (size_t)v.pitch * 8, (size_t)H->nx * 8, v.ny,
                           cudaMemcpyDeviceToDevice, s.st));
    }
    CK(cudaEventRecord(s.ev_snap, s.st));
    CK(cudaStreamWaitEvent(s.sst, s.ev_snap, 0));
    for (int k = 0; k < 4; ++k)
      if (dst[k])
        CK(cudaMemcpyAsync(dst[k] + (size_t)s.gj0 * H->nx,
                           s.snap + k * plane, plane * 8, cudaMemcpyDeviceToHost, s.sst));
    CK(cudaEventRecord(s.ev_saved, s.sst));
    s.save_issued = true;
  }
  return CSPH_OK;
}

int csph_save_wait(csph_t* H) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  for (auto& s : H->s) {
    if (!s.sst) continue;
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.sst));
  }
  return CSPH_OK;
}

int csph_get_time(csph_t* H, double* t, long long* steps_done, double* last_dt) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (!H->have_state) {
    if (t) *t = 0.0;
    if (steps_done) *steps_done = 0;
    if (last_dt) *last_dt = 0.0;
    return CSPH_OK;
  }
  Ctrl c;
  int st = read_ctrl(H, &c);
  if (st) return st;
  if (t) *t = c.t;
  if (steps_done) *steps_done = c.step;
  if (last_dt && c.step > 0) {
    Strip& s = H->s[0];
    CK(cudaMemcpy(last_dt, s.dtlog + (c.step - 1) % LOGCAP, 8, cudaMemcpyDeviceToHost));
  } else if (last_dt) {
    *last_dt = 0.0;
  }
  return CSPH_OK;
}

int csph_get_dt_log(csph_t* H, double* dt, int* limiter, int cap, int* n) {
  if (!H || cap < 0) return fail(CSPH_EINVAL, "bad argument");
  if (!H->have_state) {
    if (n) *n = 0;
    return CSPH_OK;
  }
  Ctrl c;
  int st = read_ctrl(H, &c);
  if (st) return st;
  long long done = c.step;
  long long m = done < cap ? done : cap;
  if (m > LOGCAP) m = LOGCAP;
  Strip& s = H->s[0];
  long long first = (done - m) % LOGCAP;
  long long n1 = m < LOGCAP - first ? m : LOGCAP - first;  // up to the ring end
  if (dt) {
    CK(cudaMemcpy(dt, s.dtlog + first, n1 * 8, cudaMemcpyDeviceToHost));
    if (m > n1) CK(cudaMemcpy(dt + n1, s.dtlog, (m - n1) * 8, cudaMemcpyDeviceToHost));
  }
  if (limiter) {
    CK(cudaMemcpy(limiter, s.limlog + first, n1 * 4, cudaMemcpyDeviceToHost));
    if (m > n1) CK(cudaMemcpy(limiter + n1, s.limlog, (m - n1) * 4, cudaMemcpyDeviceToHost));
  }
  if (n) *n = (int)m;
  return CSPH_OK;
}

int csph_get_maxima(csph_t* H, double M[3]) {
  if (!H || !M) return fail(CSPH_EINVAL, "bad argument");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "no state");
  Strip& s = H->s[0];
  CK(cudaSetDevice(s.dev));
  CK(cudaStreamSynchronize(s.st));
  CK(cudaMemcpy(M, s.Mlast, 3 * 8, cudaMemcpyDeviceToHost));
  return CSPH_OK;
}

// ---- load balance during a run ----

int csph_row_weights(csph_t* H, double* w) {
  if (!H || !w) return fail(CSPH_EINVAL, "bad argument");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "no state");
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    int* d = nullptr;
    CK(cudaMallocAsync((void**)&d, (size_t)s.v.ny * sizeof(int), s.st));
    if (s.v.prec == 4)
      row_wet_kernel<float><<<s.v.ny, 256, 0, s.st>>>(s.v, H->P.eps, H->host_parity, d);
    else
      row_wet_kernel<double><<<s.v.ny, 256, 0, s.st>>>(s.v, H->P.eps, H->host_parity, d);
    CK(cudaGetLastError());
    std::vector<int> cnt(s.v.ny);
    CK(cudaMemcpyAsync(cnt.data(), d, cnt.size() * sizeof(int), cudaMemcpyDeviceToHost, s.st));
    CK(cudaFreeAsync(d, s.st));
    CK(cudaStreamSynchronize(s.st));
    for (int j = 0; j < s.v.ny; ++j) w[s.gj0 + j] = (double)cnt[j] + 0.03 * (double)H->nx;
  }
  return CSPH_OK;
}

namespace {
// One field of the row migration: for every pair (old strip o, new strip r) the rows of o's
// owned range that r needs (its owned rows and, at interior edges, its 3 ghost rows),
// full padded width.  Peer copies between the strips of one process (MULTI) or NCCL
// send/recv between ranks (DIST; a rank's rows to itself by a device copy).
struct MigField {
  std::vector<char*> oldp;  // per old strip (DIST: only entry 0, this rank)
  std::vector<char*> newp;  // per new strip
  size_t es;                // element size
};

int migrate_field(csph* H, const std::vector<Strip>& olds, const std::vector<Strip>& news,
                  const std::vector<int>& ob, const std::vector<int>& nb, const MigField& f) {
  const int ny = H->ny;
  const size_t rowb = (size_t)news[0].v.pitch * f.es;
  const int nr = (int)nb.size() - 1;
  auto need = [&](int r, int* a, int* b) {  // rows [a, b) new strip r needs (global)
    *a = r > 0 ? nb[r] - GY : 0;
    *b = r < nr - 1 ? nb[r + 1] + GY : ny;
    if (*a < 0) *a = 0;
    if (*b > ny) *b = ny;
  };
  if (H->mode == MULTI) {
    for (int r = 0; r < nr; ++r) {
      const Strip& ns = news[r];
      CK(cudaSetDevice(ns.dev));
      int a, b;
      need(r, &a, &b);
      for (int o = 0; o + 1 < (int)ob.size(); ++o) {
        const int lo = a > ob[o] ? a : ob[o], hi = b < ob[o + 1] ? b : ob[o + 1];
        if (hi <= lo) continue;
        CK(cudaMemcpyPeerAsync(f.newp[r] + f.es * off(ns.v.pitch, -GX, lo - nb[r]), ns.dev,
                               f.oldp[o] + f.es * off(olds[o].v.pitch, -GX, lo - ob[o]),
                               olds[o].dev, (size_t)(hi - lo) * rowb, ns.st));
      }
    }
    return CSPH_OK;
  }
  // DIST: this rank sends the parts of its old rows every new strip needs, and receives the
  // parts of its new rows from their old owners
  const int me = H->rank;
  const Strip& ns = news[0];
  int a, b;
  need(me, &a, &b);
  NK(g_nccl.GroupStart());
  for (int o = 0; o < nr; ++o) {  // receive from old owner o
    if (o == me) continue;
    const int lo = a > ob[o] ? a : ob[o], hi = b < ob[o + 1] ? b : ob[o + 1];
    if (hi <= lo) continue;
    NK(g_nccl.Recv(f.newp[0] + f.es * off(ns.v.pitch, -GX, lo - nb[me]), (size_t)(hi - lo) * rowb,
                   ncclChar, o, H->comm, ns.st));
  }
  for (int d = 0; d < nr; ++d) {  // send to new owner d
    if (d == me) continue;
    int da, db;
    need(d, &da, &db);
    const int lo = da > ob[me] ? da : ob[me], hi = db < ob[me + 1] ? db : ob[me + 1];
    if (hi <= lo) continue;
    NK(g_nccl.Send(f.oldp[0] + f.es * off(olds[0].v.pitch, -GX, lo - ob[me]),
                   (size_t)(hi - lo) * rowb, ncclChar, d, H->comm, ns.st));
  }
  NK(g_nccl.GroupEnd());
  const int lo = a > ob[me] ? a : ob[me], hi = b < ob[me + 1] ? b : ob[me + 1];
  if (hi > lo)
    CK(cudaMemcpyAsync(f.newp[0] + f.es * off(ns.v.pitch, -GX, lo - nb[me]),
                       f.oldp[0] + f.es * off(olds[0].v.pitch, -GX, lo - ob[me]),
                       (size_t)(hi - lo) * rowb, cudaMemcpyDeviceToDevice, ns.st));
  return CSPH_OK;
}
}  // namespace

int csph_rebalance_rows(csph_t* H, const int* bounds) {
  if (!H) return fail(CSPH_EINVAL, "handle is NULL");
  if (H->mode == SINGLE) return fail(CSPH_EINVAL, "rebalance needs a DIST or MULTI handle");
  if (!H->have_state) return fail(CSPH_ENOSTATE, "no state");
  const int nr = H->nranks;
  if (check_bounds(H->ny, nr, bounds)) return CSPH_EINVAL;
  std::vector<int> nb(bounds, bounds + nr + 1), ob(nr + 1);
  // the current bounds (every rank knows them: identical on all ranks)
  if (H->mode == MULTI) {
    for (int r = 0; r < nr; ++r) ob[r] = H->s[r].gj0;
  } else {
    ob = H->bounds;
  }
  ob[nr] = H->ny;
  for (auto& s : H->s) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.st));
    CK(cudaStreamSynchronize(s.cst));
  }
  graphs_reset(H);
  const int p = H->host_parity;
  std::vector<Strip> news(H->mode == MULTI ? nr : 1);
  const bool staged = H->p.path == CSPH_PATH_STAGED;
  int st;
  for (size_t k = 0; k < news.size(); ++k) {
    const int r = H->mode == MULTI ? (int)k : H->rank;
    const int dev = H->s[k].dev;
    if ((st = strip_init(H, news[k], dev, nb[r], nb[r + 1] - nb[r], staged))) {
      for (auto& s : news) strip_free(s);
      return st;
    }
  }
  std::vector<Strip>& olds = H->s;
  const size_t es = (size_t)olds[0].v.prec;
  auto run = [&](std::function<char*(Strip&)> get, size_t esz) -> int {
    MigField f;
    f.es = esz;
    for (auto& s : olds) f.oldp.push_back(get(s));
    for (auto& s : news) f.newp.push_back(get(s));
    return migrate_field(H, olds, news, ob, nb, f);
  };
  // static fields first: allocate them on the new strips where the old ones have them
  const bool hasW = olds[0].v.W != nullptr;
  for (auto& s : news) {
    CK(cudaSetDevice(s.dev));
    const size_t n = (size_t)(s.v.ny + 2 * GY) * s.v.pitch;
    s.v.Wc = olds[0].v.Wc;
    if (hasW) {
      if ((st = dalloc(s, (void**)&s.Wbuf, n * 8))) return st;
      CK(cudaMemsetAsync(s.Wbuf, 0, n * 8, s.st));
      if (es == 4) {
        if ((st = dalloc(s, (void**)&s.Wbuf32, n * 4))) return st;
        CK(cudaMemsetAsync(s.Wbuf32, 0, n * 4, s.st));
        s.v.W = (const double*)s.Wbuf32;
      } else {
        s.v.W = s.Wbuf;
      }
    }
    double** fl[4] = {&s.cgbuf, &s.betabuf, &s.srcbuf, &s.ajbuf};
    const double* have[4] = {olds[0].cgbuf, olds[0].betabuf, olds[0].srcbuf, olds[0].ajbuf};
    for (int q = 0; q < 4; ++q)
      if (have[q]) {
        if ((st = dalloc(s, (void**)fl[q], n * 8))) return st;
        CK(cudaMemsetAsync(*fl[q], 0, n * 8, s.st));
      }
    s.v.cg = s.cgbuf; s.v.beta = s.betabuf; s.v.src = s.srcbuf; s.v.aj0 = s.ajbuf;
  }
  if (hasW) {
    if (es == 4) { if ((st = run([](Strip& s) { return (char*)s.Wbuf32; }, 4))) return st; }
    else if ((st = run([](Strip& s) { return (char*)s.Wbuf; }, 8))) return st;
  }
  if (olds[0].cgbuf && (st = run([](Strip& s) { return (char*)s.cgbuf; }, 8))) return st;
  if (olds[0].betabuf && (st = run([](Strip& s) { return (char*)s.betabuf; }, 8))) return st;
  if (olds[0].srcbuf && (st = run([](Strip& s) { return (char*)s.srcbuf; }, 8))) return st;
  if (olds[0].ajbuf && (st = run([](Strip& s) { return (char*)s.ajbuf; }, 8))) return st;
  // the current state (buffer p)
  if ((st = run([p](Strip& s) { return (char*)s.v.H[p]; }, es))) return st;
  if ((st = run([p](Strip& s) { return (char*)s.v.Qx[p]; }, es))) return st;
  if ((st = run([p](Strip& s) { return (char*)s.v.Qy[p]; }, es))) return st;
  if ((st = run([p](Strip& s) { return (char*)s.v.b[p]; }, es))) return st;
  // control block, dt log and last maxima carry over (identical on every strip / rank)
  for (size_t k = 0; k < news.size(); ++k) {
    Strip& s = news[k];
    const Strip& o = olds[H->mode == MULTI ? 0 : k];
    CK(cudaSetDevice(s.dev));
    CK(cudaMemcpyPeerAsync(s.ctrl, s.dev, o.ctrl, o.dev, sizeof(Ctrl), s.st));
    CK(cudaMemcpyPeerAsync(s.dtlog, s.dev, o.dtlog, o.dev, LOGCAP * sizeof(double), s.st));
    CK(cudaMemcpyPeerAsync(s.limlog, s.dev, o.limlog, o.dev, LOGCAP * sizeof(int), s.st));
    CK(cudaMemcpyPeerAsync(s.Mlast, s.dev, o.Mlast, o.dev, 4 * sizeof(double), s.st));
    // wall ghosts of the state buffer and of the static fields (interior edges: migrated)
    launch_mirror(s.v, s.ctrl, 0, s.st, &H->launches);
    for (double* F : {s.cgbuf, s.betabuf, s.srcbuf, s.ajbuf}) {
      if (!F) continue;
      int n1 = (s.v.ny + 2 * GY) * 6, n2 = (s.v.nx + 6) * 6;
      mirror_field_kernel<<<(n1 + 255) / 256, 256, 0, s.st>>>(s.v, F);
      mirror_field_y_kernel<<<(n2 + 255) / 256, 256, 0, s.st>>>(s.v, F);
    }
    CK(cudaGetLastError());
    if (s.auto_ty && H->p.path == CSPH_PATH_FUSED && (st = choose_tile_rows(H, s, p))) return st;
    if ((st = order_reset(H, s))) return st;
    CK(cudaStreamSynchronize(s.st));
  }
  // a caller stream (csph_set_stream, single-strip handles) carries over
  if (H->s.size() == 1 && !H->s[0].own_stream) {
    CK(cudaSetDevice(news[0].dev));
    CK(cudaStreamDestroy(news[0].st));
    news[0].st = H->s[0].st;
    news[0].own_stream = false;
  }
  for (auto& s : H->s) strip_free(s);
  H->s = std::move(news);
  if (H->mode == MULTI) push_link_multi(H);
  if (H->mode == DIST) ipc_unlink(H);  // new buffers: the caller links them again
  if (H->mode == DIST) H->bounds = nb;
  return CSPH_OK;
}

}  // extern "C"
