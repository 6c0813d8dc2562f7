// Dev probe: DFMA vs DMMA (mma.sync m8n8k4 f64) throughput and overlap on B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>  // 0 dfma only, 1 dmma only, 2 both
__global__ void k(double* out, int iters, double x) {
  double f[8]; double c[8][2];
  for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x + i; c[i][0] = c[i][1] = i; }
  double a = x * threadIdx.x, b = x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(f[i], x, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += f[i] + c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks_per_sm : {4, 8}) for (int mode = 0; mode < 3; ++mode) {
    int iters = 20000; float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<sms * blocks_per_sm, 256>>>(o, iters, 0.999);
      if (mode == 1) k<1><<<sms * blocks_per_sm, 256>>>(o, iters, 0.999);
      if (mode == 2) k<2><<<sms * blocks_per_sm, 256>>>(o, iters, 0.999);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double threads = (double)sms * blocks_per_sm * 256;
    double dfma_flop = (mode != 1) ? 2.0 * 8 * iters * threads : 0;
    double dmma_flop = (mode != 0) ? 8.0 * iters * (threads / 32) * 2 * 256 : 0;
    printf("bpsm %d mode %d: %.3f ms  DFMA %.2f TF  DMMA %.2f TF  total %.2f TF  err=%s\n", blocks_per_sm, mode, ms,
           dfma_flop / ms / 1e9, dmma_flop / ms / 1e9, (dfma_flop + dmma_flop) / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
