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

// Fused y-marching step (csph_fused.cu). Rows [row0, row1) of the strip.
void launch_fused_step(const StripView& S, Ctrl* C, const Phys& P, unsigned long long* gM,
                       int row0, int row1, int tile_rows, cudaStream_t st, long long* nlaunch);

// Service kernels (csph_api.cu).
void launch_mirror(const StripView& S, const Ctrl* C, int next_parity_from_ctrl,
                   cudaStream_t st, long long* nlaunch);

}  // namespace ck
