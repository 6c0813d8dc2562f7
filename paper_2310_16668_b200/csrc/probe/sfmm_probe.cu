// Measurement and test hooks (include/sfmm_probe.h), built as their own
// library: NOT part of the drop-in apply ABI.
//   * FP64 pipe probe: the roofline denominator for the FP64-bound
//     translation kernel (MEASURED_PEAKS.json carries only HBM and bf16 peaks);
//   * device-math checks of the product's table-driven log / sincos
//     (fastmath.cuh) against the CUDA library.
#include <cuda_runtime.h>

#include <algorithm>

#include "fastmath.cuh"
#include "sfmm_probe.h"

namespace sfmm_gpu {
namespace {

__global__ void sincos_check(const double* x, int64_t n, const double2* tab, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s, c, st, ct, s_ref, c_ref;
    sincos_fast(x[i], &s, &c);
    sincos_tab_scaled(tab, x[i], 1.0, &ct, &st);
    sincos(x[i], &s_ref, &c_ref);
    out[6 * i] = s;
    out[6 * i + 1] = c;
    out[6 * i + 2] = st;
    out[6 * i + 3] = ct;
    out[6 * i + 4] = s_ref;
    out[6 * i + 5] = c_ref;
  }
}

}  // namespace

namespace {
__global__ void log_check(const double* x, int64_t n, const double* tab, double* out) {
  __shared__ __align__(16) double lt[kLogTabLen];
  for (int i = threadIdx.x; i < kLogTabLen; i += blockDim.x) lt[i] = tab[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[2 * i] = log_tab(log_tab_addr(lt), x[i]);
    out[2 * i + 1] = log(x[i]);
  }
}
}  // namespace

namespace {

int test_log(const double* x_host, int64_t n, double* out_host) {
  double *dx = nullptr, *dout = nullptr, *dtab = nullptr;
  double tab[kLogTabLen];
  fill_log_table(tab);
  int rc = -1;
  if (cudaMalloc(&dx, std::max<int64_t>(n, 1) * sizeof(double)) == cudaSuccess &&
      cudaMalloc(&dout, std::max<int64_t>(2 * n, 1) * sizeof(double)) == cudaSuccess &&
      cudaMalloc(&dtab, sizeof(tab)) == cudaSuccess) {
    cudaMemcpy(dx, x_host, n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(dtab, tab, sizeof(tab), cudaMemcpyHostToDevice);
    log_check<<<148 * 4, 256>>>(dx, n, dtab, dout);
    cudaMemcpy(out_host, dout, 2 * n * sizeof(double), cudaMemcpyDeviceToHost);
    rc = cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  cudaFree(dx);
  cudaFree(dout);
  cudaFree(dtab);
  return rc;
}

int test_sincos(const double* x_host, int64_t n, double* out_host) {
  double *dx = nullptr, *dout = nullptr;
  double2* dtab = nullptr;
  double2 tab[kSinCosTab];
  fill_sincos_table(tab);
  if (cudaMalloc(&dx, n * sizeof(double)) != cudaSuccess) return -1;
  if (cudaMalloc(&dout, 6 * n * sizeof(double)) != cudaSuccess) return -1;
  if (cudaMalloc(&dtab, sizeof(tab)) != cudaSuccess) return -1;
  cudaMemcpy(dx, x_host, n * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(dtab, tab, sizeof(tab), cudaMemcpyHostToDevice);
  sincos_check<<<148 * 4, 256>>>(dx, n, dtab, dout);
  cudaMemcpy(out_host, dout, 6 * n * sizeof(double), cudaMemcpyDeviceToHost);
  const bool ok = cudaGetLastError() == cudaSuccess;
  cudaFree(dx);
  cudaFree(dout);
  cudaFree(dtab);
  return ok ? 0 : -1;
}

namespace {

constexpr int kChains = 8;

// One multiplicand comes from a uniform register (the kernel parameter) and the
// addend from a per-thread register, so the loop is not limited by register-
// file read bandwidth (three 64-bit register operands per DFMA measure ~92 %).
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b0) {
  double x[kChains];
  const double b = b0 * (threadIdx.x + 1);
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the loop alive
}

}  // namespace

double measure_fp64_peak(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 4 CTAs x 256 threads per SM, 8 independent chains each: 37.0 TFLOP/s at
  // 1965 MHz on B200 (64 DFMA/clk/SM); ~13 ms per launch so the clocks settle
  const int blocks = sms * 4, threads = 256;
  const int iters = 200000;
  float ms = 0;
  dfma_loop<<<blocks, threads>>>(out, iters / 10, 0.999999, 1e-7);  // warm-up
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * kChains * (double)iters * blocks * threads;
    best = std::max(best, flop / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1;
}

}  // namespace
}  // namespace sfmm_gpu

extern "C" {

int sfmm_probe_test_log(const double* x, int64_t n, double* out) {
  if (!x || !out || n < 0) return 1;
  return sfmm_gpu::test_log(x, n, out) == 0 ? 0 : 3;
}

int sfmm_probe_test_sincos(const double* x, int64_t n, double* out) {
  if (!x || !out || n < 0) return 1;
  return sfmm_gpu::test_sincos(x, n, out) == 0 ? 0 : 3;
}

int sfmm_probe_fp64_peak(int device, double* tflops) {
  if (!tflops) return 1;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  *tflops = sfmm_gpu::measure_fp64_peak(device);
  if (prev >= 0) cudaSetDevice(prev);
  return *tflops > 0 ? 0 : 3;
}

}  // extern "C"
