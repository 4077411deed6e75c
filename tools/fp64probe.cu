// fp64 pipe probe (dev aid): latency of dependent DFMA/DADD chains and throughput with
// ILP 1..8 at several warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps_per_sm, int nsm) {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
  const int n = 4096;
  int threads = 32 * warps_per_sm;
  if (threads > 1024) threads = 1024;
  int blocks = nsm * (32 * warps_per_sm / threads);
  chain<ILP><<<blocks, threads>>>(out, 0.999, 1e-3, n, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<ILP><<<blocks, threads>>>(out, 0.999, 1e-3, n, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)blocks * threads * n * ILP;
  printf("ILP %d warps/SM %2d: %.1f cyc per dependent DFMA, %.2f T DFMA/s (%.1f lanes/clk/SM at 1.9GHz)\n",
         ILP, warps_per_sm, (double)c / n, ops / ms / 1e9, ops / ms / 1e3 / 1.9e9 / nsm * 1e3 / 1e3);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {1, 4, 8, 12, 16, 32}) run<1>(w, nsm);
  for (int w : {4, 8, 12, 16}) run<2>(w, nsm);
  for (int w : {4, 8, 12, 16}) run<4>(w, nsm);
  for (int w : {4, 8, 12}) run<8>(w, nsm);
  return 0;
}
