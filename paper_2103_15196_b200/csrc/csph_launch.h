// csph_launch.h -- internal interfaces between the C-ABI layer and the kernels.
#pragma once

#include "csph_internal.cuh"

namespace ck {

// HBM intermediates of the staged (paper K1..K8) path, padded layout.
struct Scratch {
  double *eta, *r, *u, *v, *phix, *phiy, *gam, *Hh, *ut, *vt, *phix2, *phiy2;
  double *QLx, *QLy, *J0x, *J0y, *J0a;
  double *FH, *FQx, *FQy, *FJ, *GH, *GQx, *GQy, *GJ;
  unsigned char* w;
};

void launch_staged_step(const StripView& S, Ctrl* C, const Scratch& T, const Phys& P,
                        unsigned long long* gM, cudaStream_t st, long long* nlaunch);

// HGS tile flags of the fused path: a tile is the TX x TY chunk
// one CTA marches.  fprev/fnext: band masks (HGS_*) of the tile's wet output cells for
// the previous / this step; tstate: consecutive identity copies of the tile (2 = both
// ping-pong buffers hold the same values, the tile may be skipped outright).
// Band bits of a tile flag: some output cell wet anywhere / in the first row / the last
// row / the first column / the last column of the tile.
enum : unsigned { HGS_ANY = 1, HGS_TOP = 2, HGS_BOT = 4, HGS_LEFT = 8, HGS_RIGHT = 16, HGS_ALL = 31 };

struct Hgs {
  const unsigned char* fprev;
  unsigned char* fnext;
  // flags of the facing tile row of the neighbouring strips (previous step), [ntx] each;
  // nullptr on a global edge.  Filled by the halo exchange with the halo rows.
  const unsigned char* glo;
  const unsigned char* ghi;
  unsigned char* tstate;
  int ntx, nty;
  int enable;
  unsigned long long* stats;  // [0] tiles marched, [1] copied (identity), [2] skipped
  // Launch order: CTA i of the launch takes tile order[i] (linear index
  // within the launch's tile rows; nullptr = natural order), costliest first.  cost[ti]:
  // the rows the tile's march computed at full cost (0 for identity / skipped tiles),
  // written by the step kernel; the order of the step after next is sorted from it.
  const int* order;
  unsigned short* cost;
};

#ifndef CSPH_NT
#define CSPH_NT 128   // threads per CTA of the fused kernel (development knob)
#endif
#ifndef CSPH_MINB
#define CSPH_MINB 3   // resident fp64 CTAs per SM (development knob, with CSPH_NT)
#endif
constexpr int FUSED_NT = CSPH_NT;
constexpr int FUSED_TX = CSPH_NT - 8;  // output columns per CTA of the fused kernel (NT - 8)
constexpr int FUSED_MINB = CSPH_MINB;
static_assert(FUSED_NT % 32 == 0 && FUSED_NT >= 64 && FUSED_NT <= 1024, "CTA width: whole warps");

// Fused y-marching step (csph_fused.cu). Rows [row0, row1) of the strip; row0 must be
// a multiple of tile_rows when HGS is enabled.
void launch_fused_step(const StripView& S, Ctrl* C, const Phys& P, unsigned long long* gM,
                       int row0, int row1, int tile_rows, const Hgs& hgs, cudaStream_t st,
                       long long* nlaunch);

// Order the tiles of tile rows [tr0, tr1) by descending cost into order[0, ntx (tr1 - tr0))
// (one CTA, a counting sort; ties in any order: the step's results do not depend on it).
void launch_order_tiles(const unsigned short* cost, int ntx, int tr0, int tr1, int* order,
                        cudaStream_t st, long long* nlaunch);

// order[i] = i for i < n (the natural order).
void launch_order_identity(int* order, int n, cudaStream_t st, long long* nlaunch);

// Service kernels (csph_api.cu).
void launch_mirror(const StripView& S, const Ctrl* C, int next_parity_from_ctrl,
                   cudaStream_t st, long long* nlaunch);

}  // namespace ck
