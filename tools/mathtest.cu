#include <cstdio>
#include "/root/repo/paper_2103_15196_b200/csrc/csph_internal.cuh"
using namespace ck;
__global__ void k(long long n, unsigned long long seed, unsigned long long* bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long st = (long long)gridDim.x * blockDim.x;
  unsigned long long nb = 0;
  for (; i < n; i += st) {
    unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    // exponent in [-200, 200], random mantissa
    unsigned long long e = 1023 - 200 + (z >> 52) % 401;
    double x = __longlong_as_double((long long)((e << 52) | (z & 0xFFFFFFFFFFFFFull)));
    if (rcp_nb(x) != 1.0 / x) nb++;
    if (sqrt_nb(x) != sqrt(x)) nb++;
  }
  atomicAdd(bad, nb);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  k<<<4096, 256>>>(1ll << 32, 12345, d);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mismatches %llu of 2^32 x 2\n", h);
}
