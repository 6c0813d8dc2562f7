#include <cstdio>
#include <cuda_runtime.h>
template <int V> __device__ __forceinline__ double seed(double r2) {
  double y;
  if (V == 0) asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  else if (V == 1) y = fma(r2, -0.5, 1.5);            // FP64 op instead of MUFU
  else { float f = rsqrtf((float)r2); y = (double)f; } // FP32 MUFU + converts
  return y;
}
template <int V, int R>
__global__ void k(double* out, int iters, double step) {
  double x[R], y[R], z[R], au[R];
  for (int r = 0; r < R; ++r) { x[r] = 0.1 * threadIdx.x + r; y[r] = 0.2 * r; z[r] = 0.3; au[r] = 0; }
  double sx = 0.5, sy = 0.25, sz = 0.125, q = 1.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = x[r] - sx, dy = y[r] - sy, dz = z[r] - sz;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double yy = seed<V>(r2);
      const double e = fma(-r2, yy * yy, 1.0);
      au[r] = fma(fma(fma(0.375, e, 0.5), yy * e, yy), q, au[r]);
    }
    sx += step; sy -= step; sz += step; q = -q;
  }
  double s = 0; for (int r = 0; r < R; ++r) s += au[r];
  if (s == 1.2345) out[0] = s;
}
template <int V, int R> void run(int bpsm) {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<V, R><<<sms * bpsm, 128>>>(o, iters, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  double pairs = (double)sms * bpsm * 128 * iters * R;
  double fp64 = pairs * (V == 1 ? 13.0 : 12.0);
  printf("V=%d R=%d warps/SMSP=%d: %.3e pairs/s, FP64 instr %.1f%% of 64/clk/SM@1965\n", V, R, bpsm,
         pairs / ms * 1e3, 100.0 * fp64 / (ms * 1e-3) / (64.0 * sms * 1.965e9));
}
int main() {
  run<0, 4>(4); run<1, 4>(4); run<2, 4>(4);
  run<0, 4>(8); run<1, 4>(8); run<2, 4>(8);
  return 0;
}
