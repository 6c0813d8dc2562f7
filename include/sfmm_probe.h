/*
 * sfmm_probe.h -- measurement and test hooks (lib/libsfmm_probe.so).
 *
 * NOT part of the drop-in apply ABI (include/sfmm_gpu.h): a separate library
 * that bench.py loads for its roofline denominator and tests/ load to check
 * the device math the apply kernels use.  Return 0 on success, 1 on a bad
 * argument, 3 on a CUDA failure (the sfmm_gpu.h codes).
 */
#ifndef SFMM_PROBE_H_
#define SFMM_PROBE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Measured FP64 FMA throughput of the device (TFLOP/s, 2 flop per DFMA), from
 * a register-resident DFMA loop run on every SM (best of 5 launches of ~13 ms). */
int sfmm_probe_fp64_peak(int device, double* tflops);

/* out[6i..6i+5] = (sin, cos) of x_i from the branch-free routine, the
 * table-driven routine of the Helmholtz kernels (fastmath.cuh) and the CUDA
 * library, on the current device. */
int sfmm_probe_test_sincos(const double* x, int64_t n, double* out);

/* out[2i], out[2i+1] = log(x_i) from the table-driven routine of the
 * Laplace-2D kernels (fastmath.cuh) and from the CUDA library. */
int sfmm_probe_test_log(const double* x, int64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* SFMM_PROBE_H_ */
