// Structured hard cases for the branch-free reciprocal / square root (dev aid, GPU):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/mt tools/mathtest.cu && /tmp/mt
// Mantissas near all-ones, near zero, all-ones with one bit cleared, a run of top ones over a
// random tail, each over exponents [-300, 300]; prints the first failing operands.
#include <cstdio>
#include "../paper_2103_15196_b200/csrc/csph_internal.cuh"
using namespace ck;

__device__ unsigned long long mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k(long long n, unsigned long long* bad, double* first) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long st = (long long)gridDim.x * blockDim.x;
  const unsigned long long ONES = 0xFFFFFFFFFFFFFull;
  for (; i < n; i += st) {
    const unsigned long long z = mix(0x1234567ull + (unsigned long long)i * 0x9E3779B97F4A7C15ull);
    const unsigned long long e = 1023 - 300 + (z >> 52) % 601;
    unsigned long long m;
    switch (i & 3) {
      case 0: m = ONES - ((unsigned long long)(i >> 2) & 4095); break;
      case 1: m = (unsigned long long)(i >> 2) & 4095; break;
      case 2: m = ONES ^ (1ull << ((i >> 2) % 52)); break;
      default: {
        const int s = (int)((i >> 2) % 52);
        m = ((ONES << s) & ONES) | (z & ((1ull << s) - 1));
      }
    }
    const double x = __longlong_as_double((long long)((e << 52) | m));
    int which = 0;
    if (rcp_nb(x) != 1.0 / x) which = 1;
    else if (sqrt_nb(x) != sqrt(x)) which = 2;
    else if (sqrt0nb(x) != sqrt(x)) which = 3;
    if (which) {
      atomicAdd(&bad[which], 1ull);
      const bool allones = m == ONES;
      atomicAdd(&bad[4 + (allones ? 1 : 0)], 1ull);
      if (!allones) {
        const unsigned long long k2 = atomicAdd(bad, 1ull);
        if (k2 < 8) { first[2 * k2] = x; first[2 * k2 + 1] = which; }
      }
    }
  }
}

int main() {
  unsigned long long* d; double* f;
  cudaMalloc(&d, 8 * 8); cudaMemset(d, 0, 8 * 8); cudaMalloc(&f, 16 * 8);
  const long long n = 1ll << 30;
  k<<<4096, 256>>>(n, d, f);
  unsigned long long hb[8]; double hf[16];
  cudaMemcpy(hb, d, 64, cudaMemcpyDeviceToHost); cudaMemcpy(hf, f, 16 * 8, cudaMemcpyDeviceToHost);
  const unsigned long long h = hb[0];
  printf("of %lld structured operands: rcp %llu, sqrt %llu, sqrt0 %llu mismatches; all-ones mantissa %llu, "
         "other %llu\n", n, hb[1], hb[2], hb[3], hb[5], hb[4]);
  for (int j = 0; j < 8 && j < (int)h; ++j) printf("  x = %a  (%s)\n", hf[2 * j], hf[2 * j + 1] == 1 ? "rcp" : hf[2 * j + 1] == 2 ? "sqrt" : "sqrt0");
}
