// Accuracy of rsqrt variants for the Laplace-3D translation kernel (dev tool).
//   a: MUFU.RSQ64H seed + one Newton step (3 FP64 ops after the seed)
//   b: MUFU.RSQ64H seed + cubic correction (the production exact path)
// Prints the max / mean relative error of (a) over log-uniform inputs, per
// exponent parity, and for a dense mantissa sweep (the bias constant).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

__device__ double seed64(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  return y;
}
__global__ void run(const double* x, int n, double* a, double* b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r2 = x[i];
  const double y = seed64(r2);
  const double e = fma(-r2, y * y, 1.0);
  a[i] = fma(0.5 * y, e, y);
  b[i] = fma(fma(0.375, e, 0.5), y * e, y);
}
int main() {
  const int n = 1 << 24;
  std::vector<double> x(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int i = 0; i < n / 2; ++i) x[i] = std::exp2(-40.0 + 80.0 * u(g));     // log-uniform
  for (int i = n / 2; i < n; ++i) x[i] = 1.0 + 3.0 * (double)(i - n / 2) / (n / 2);  // [1,4) sweep
  double *dx, *da, *db;
  cudaMalloc(&dx, n * 8); cudaMalloc(&da, n * 8); cudaMalloc(&db, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  run<<<(n + 255) / 256, 256>>>(dx, n, da, db);
  std::vector<double> a(n), b(n);
  cudaMemcpy(a.data(), da, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), db, n * 8, cudaMemcpyDeviceToHost);
  for (int part = 0; part < 2; ++part) {
    long double mx = 0, mean = 0, mxb = 0, lw = 0, lmean = 0;
    int i0 = part ? n / 2 : 0, i1 = part ? n : n / 2;
    for (int i = i0; i < i1; ++i) {
      long double ex = 1.0L / sqrtl((long double)x[i]);
      long double ra = (a[i] - ex) / ex, rb = (b[i] - ex) / ex;
      mx = fmaxl(mx, fabsl(ra));
      mxb = fmaxl(mxb, fabsl(rb));
      mean += ra;
      // log-uniform weight for the [1,4) sweep: density 1/m
      long double w = 1.0L / x[i];
      lw += w;
      lmean += w * ra;
    }
    printf("%s: newton max %.3Le mean %.3Le (1/m-weighted mean %.3Le) | cubic max %.3Le\n",
           part ? "sweep[1,4)" : "loguniform", mx, mean / (i1 - i0), lmean / lw, mxb);
  }
  return 0;
}
