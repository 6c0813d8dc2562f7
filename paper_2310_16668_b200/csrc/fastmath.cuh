// Branch-free FP64 sincos for the Helmholtz kernel, |x| <= 2^20.
//
// kappa * r stays small in every configuration (kappa = 10, r <= sqrt(3) in
// the unit cube), so the general library sincos -- which keeps a Payne-Hanek
// slow path behind a branch -- does more work than needed.  Here: Cody-Waite
// reduction by pi/2 in three FMA steps (fdlibm's pio2_1/pio2_2/pio2_2t split,
// exact for |j| < 2^20), then the fdlibm __kernel_sin / __kernel_cos minimax
// polynomials on |t| <= pi/4 (< 1 ulp), then the quadrant swap.  About 22
// FP64 instructions.  Checked against the CUDA math library in
// tests/test_kernels_gpu.py.
#pragma once

namespace sfmm_gpu {

__device__ __forceinline__ void sincos_fast(double x, double* sp, double* cp) {
  const double j = rint(x * 0.63661977236758134308);  // 2/pi
  double t = fma(-j, 1.57079632673412561417e+00, x);
  t = fma(-j, 6.07710050630396597660e-11, t);
  t = fma(-j, 2.02226624879595063154e-21, t);
  const double z = t * t;
  // sin(t) = t + t^3 (S1 + z S2 + ... + z^5 S6)
  double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  ps = fma(z, ps, 2.75573137070700676789e-06);
  ps = fma(z, ps, -1.98412698298579493134e-04);
  ps = fma(z, ps, 8.33333333332248946124e-03);
  ps = fma(z, ps, -1.66666666666666324348e-01);
  const double s = fma(t * z, ps, t);
  // cos(t) = 1 - z/2 + z^2 (C1 + z C2 + ... + z^5 C6), fdlibm's error-compensated form
  double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  pc = fma(z, pc, -2.75573143513906633035e-07);
  pc = fma(z, pc, 2.48015872894767294178e-05);
  pc = fma(z, pc, -1.38888888888741095749e-03);
  pc = fma(z, pc, 4.16666666666666019037e-02);
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double c = w + (((1.0 - w) - hz) + z * z * pc);
  const int q = static_cast<int>(static_cast<long long>(j) & 3);
  const double sv = (q & 1) ? c : s;
  const double cv = (q & 1) ? s : c;
  *sp = (q & 2) ? -sv : sv;
  *cp = ((q + 1) & 2) ? -cv : cv;
}

}  // namespace sfmm_gpu
