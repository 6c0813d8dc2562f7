// Dev probe: throughput of the Laplace-3D pair chain (13 FP64 ops + MUFU) with
// R rows per thread and W warps per SMSP, no memory traffic.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rs(double r2) {
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double e = fma(-r2, y * y, 1.0);
  return fma(fma(0.375, e, 0.5), y * e, y);
}
template <int R>
__global__ void k(double* out, int iters, double step) {
  double x[R], y[R], z[R], au[R];
  for (int r = 0; r < R; ++r) { x[r] = 0.1 * threadIdx.x + r; y[r] = 0.2 * r; z[r] = 0.3; au[r] = 0; }
  double sx = 0.5, sy = 0.25, sz = 0.125, q = 1.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = x[r] - sx, dy = y[r] - sy, dz = z[r] - sz;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      au[r] = fma(rs(r2), q, au[r]);
    }
    sx += step; sy -= step; sz += step; q = -q;
  }
  double s = 0; for (int r = 0; r < R; ++r) s += au[r];
  if (s == 1.2345) out[0] = s;
}
template <int R> void run(int bpsm, int threads) {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<R><<<sms * bpsm, threads>>>(o, iters, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  double pairs = (double)sms * bpsm * threads * iters * R;
  // 3 DADD + DMUL + 2 DFMA + (DMUL, DFMA, DFMA, DMUL, DFMA) + DFMA = 12 FP64 + 3 DADD for sx.. per it/R
  double fp64 = pairs * 12.0;
  printf("R=%d warps/SMSP=%d: %.3e pairs/s, %.1f%% of FP64 instr peak (64/clk/SM @1965)\n", R, bpsm * threads / 32 / 4,
         pairs / ms * 1e3, 100.0 * fp64 / (ms * 1e-3) / (64.0 * sms * 1.965e9));
}
int main() {
  run<1>(4, 128); run<2>(4, 128); run<4>(4, 128); run<8>(4, 128);
  run<1>(8, 128); run<2>(8, 128); run<4>(8, 128);
  run<4>(2, 128); run<4>(3, 128);
  return 0;
}
