// Multi-right-hand-side apply (nrhs > 1): K0m, K1m, K2m, K3m, K4m.
//
// The reference applies one right-hand side per call (apply.hpp:91-94); a
// user with 16 charge vectors runs fmm_apply 16 times and regenerates every
// kernel entry 16 times.  Here the right-hand sides go through the tree
// together, 16 at a time, so each G(x_i, x_j) is generated once and applied to
// all of them: the translation step becomes a generated-matrix x (n_c x 16)
// product issued on the FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA).
//
// K2m task = 16 target rows (two 8-row DMMA tiles).  Per k-step (4 sources)
// every lane generates the one G entry its A-fragment holds (row = lane/4,
// source = lane%4) -- exactly one pair per lane, no shuffles -- and the warp
// issues 8 DMMAs (complex) or 2 (real) per row tile.  Complex products use
// U = Gr [Ar | Ai] + Gi [-Ai | Ar] so both real products accumulate into the
// same fragments.  On B200 DMMA shares the FP64 datapath with DFMA (both
// measured at 37 TFLOP/s, see profiles/), so the gain over scalar code is
// issue slots and registers, not peak.
#include <math.h>

#include <algorithm>

#include "launch.h"

namespace sfmm_gpu {
namespace {

constexpr int kMWarps = 4;
constexpr int kMThreads = 32 * kMWarps;
constexpr int kChunk = 16;  // sources staged per chunk (4 k-steps of 4)
constexpr double kInv4Pi = 0.0795774715459476678844418816862571810;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double rsqrt_fp64m(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double e = fma(-r2, y * y, 1.0);
  return fma(fma(0.375, e, 0.5), y * e, y);
}

struct K2MArgs {
  const BoxRec* box;
  const EntryRange* er;
  const int32_t* ent;
  const Task* tasks;
  int64_t n_tasks;
  const double *X, *Y, *Z;
  const int32_t* sid;
  const double* Q;   // [slot][kNRHS] scalars (complex: interleaved)
  const double* QH;  // [skel][kNRHS]
  double* U;
  double* UH;
  int* counter;
  int* err;
  double kappa;
};

template <bool CPLX>
struct WarpSmemM {
  static constexpr int SW = CPLX ? 2 : 1;
  double x[kChunk], y[kChunk], z[kChunk];
  double a[kChunk][kNRHS * SW];
  double h[kChunk][kNRHS * SW];
};

__device__ __noinline__ void verify_row_m(const K2MArgs& a, int32_t b, int32_t row, int dim) {
  const BoxRec tb = a.box[b];
  const int64_t s = tb.slot + row;
  const double x = a.X[s], y = a.Y[s], z = a.Z[s];
  const int32_t id = a.sid[s];
  const EntryRange er = a.er[b];
  for (int e = 0; e < er.count; ++e) {
    const BoxRec sb = a.box[a.ent[er.begin + e] >> kModeBits];
    for (int j = 0; j < sb.n; ++j) {
      const int64_t t = sb.slot + j;
      const double dx = x - a.X[t], dy = y - a.Y[t], dz = dim == 3 ? z - a.Z[t] : 0.0;
      const double r2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (r2 == 0.0 && a.sid[t] != id) atomicOr(a.err, 1);
    }
  }
}

// KER: 0 laplace2d, 1 laplace3d, 3 helmholtz3d
template <int KER>
__global__ void __launch_bounds__(kMThreads, 3) k2m_translate(K2MArgs a) {
  constexpr bool CPLX = KER == SFMM_HELMHOLTZ3D;
  constexpr int SW = CPLX ? 2 : 1;
  constexpr int NB = CPLX ? 4 : 2;  // 8-column DMMA blocks across [Ur | Ui] or [U]
  constexpr int DIM = KER == SFMM_LAPLACE2D ? 2 : 3;
  __shared__ WarpSmemM<CPLX> smem[kMWarps];
  WarpSmemM<CPLX>& sm = smem[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int rq = lane >> 2, kq = lane & 3;  // A-fragment row / k index of this lane
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.counter, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.n_tasks) return;
    const Task task = a.tasks[t];
    const BoxRec tb = a.box[task.box];
    double xr[2], yr[2], zr[2];
    int rowi[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = task.row0 + mt * 8 + rq;
      rowi[mt] = row;
      const int64_t s = tb.slot + (row < task.row0 + task.nrows ? row : task.row0);
      xr[mt] = a.X[s];
      yr[mt] = a.Y[s];
      zr[mt] = DIM == 3 ? a.Z[s] : 0.0;
    }
    double C[2][NB][2], H[2][NB][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) C[mt][nb][0] = C[mt][nb][1] = H[mt][nb][0] = H[mt][nb][1] = 0.0;
    const bool skel_rows = task.row0 < tb.k;
    const EntryRange er = a.er[task.box];
    for (int e = 0; e < er.count; ++e) {
      const int32_t code = a.ent[er.begin + e];
      const int32_t c = code >> kModeBits;
      const int mode = code & kModeMask;
      const BoxRec sb = a.box[c];
      const bool self = c == task.box;
      for (int j0 = 0; j0 < sb.n; j0 += kChunk) {
        // stage 16 sources: coordinates + per-mode weights for all rhs
        __syncwarp();
        if (lane < kChunk) {
          const int j = j0 + lane;
          if (j < sb.n) {
            const int64_t s = sb.slot + j;
            sm.x[lane] = a.X[s];
            sm.y[lane] = a.Y[s];
            sm.z[lane] = DIM == 3 ? a.Z[s] : 0.0;
          } else {
            // far away, zero weight; moderate so sincos(kappa r) stays on its
            // fast argument-reduction path
            sm.x[lane] = sm.y[lane] = sm.z[lane] = 1e3;
          }
        }
        for (int v = lane; v < kChunk * kNRHS * SW; v += 32) {
          const int jj = v / (kNRHS * SW), col = v % (kNRHS * SW);
          const int j = j0 + jj;
          double q = 0.0, qh = 0.0;
          if (j < sb.n) {
            q = a.Q[(sb.slot + j) * (kNRHS * SW) + col];
            if (j < sb.k) qh = a.QH[(sb.skel + j) * (kNRHS * SW) + col];
          }
          double wa = q, wh = 0.0;
          if (mode == kIFO) wh = qh;
          else if (mode == kIFS) wh = q;
          else if (mode == kTFO) wa = q - qh;
          sm.a[jj][col] = wa;
          sm.h[jj][col] = wh;
        }
        __syncwarp();
        const bool need_h = skel_rows && (mode == kIFS || (mode == kIFO && j0 < sb.k));
#pragma unroll
        for (int ks = 0; ks < kChunk; ks += 4) {
          const int js = ks + kq;  // this lane's source within the chunk
          double gr[2], gi[2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const double dx = xr[mt] - sm.x[js], dy = yr[mt] - sm.y[js];
            double r2 = fma(dy, dy, dx * dx);
            if (DIM == 3) {
              const double dz = zr[mt] - sm.z[js];
              r2 = fma(dz, dz, r2);
            }
            if (KER == SFMM_LAPLACE2D) {
              gr[mt] = log(r2);
              gi[mt] = 0.0;
            } else {
              const double yv = rsqrt_fp64m(r2);
              if (CPLX) {
                double sn, cs;
                sincos(a.kappa * (r2 * yv), &sn, &cs);
                gr[mt] = cs * yv;
                gi[mt] = sn * yv;
              } else {
                gr[mt] = yv;
                gi[mt] = 0.0;
              }
            }
            if (self && rowi[mt] == j0 + js) gr[mt] = gi[mt] = 0.0;
          }
          // B fragments: source js, rhs columns rq and 8 + rq
          double b1[NB], b2[NB], h1[NB], h2[NB];
          if (CPLX) {
            const double ar0 = sm.a[js][2 * rq], ai0 = sm.a[js][2 * rq + 1];
            const double ar8 = sm.a[js][2 * (8 + rq)], ai8 = sm.a[js][2 * (8 + rq) + 1];
            b1[0] = ar0; b1[1] = ar8; b1[2] = ai0; b1[3] = ai8;
            b2[0] = -ai0; b2[1] = -ai8; b2[2] = ar0; b2[3] = ar8;
            if (need_h) {
              const double hr0 = sm.h[js][2 * rq], hi0 = sm.h[js][2 * rq + 1];
              const double hr8 = sm.h[js][2 * (8 + rq)], hi8 = sm.h[js][2 * (8 + rq) + 1];
              h1[0] = hr0; h1[1] = hr8; h1[2] = hi0; h1[3] = hi8;
              h2[0] = -hi0; h2[1] = -hi8; h2[2] = hr0; h2[3] = hr8;
            }
          } else {
            b1[0] = sm.a[js][rq];
            b1[1] = sm.a[js][8 + rq];
            if (need_h) {
              h1[0] = sm.h[js][rq];
              h1[1] = sm.h[js][8 + rq];
            }
          }
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              dmma(C[mt][nb][0], C[mt][nb][1], gr[mt], b1[nb]);
              if (CPLX) dmma(C[mt][nb][0], C[mt][nb][1], gi[mt], b2[nb]);
            }
          if (need_h) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int nb = 0; nb < NB; ++nb) {
                dmma(H[mt][nb][0], H[mt][nb][1], gr[mt], h1[nb]);
                if (CPLX) dmma(H[mt][nb][0], H[mt][nb][1], gi[mt], h2[nb]);
              }
          }
        }
      }
    }
    // epilogue: lane holds rows rq (+8) and rhs columns c0, c0+1, 8+c0, 9+c0
    const double scale = CPLX ? 0.25 : (KER == SFMM_LAPLACE3D ? kInv4Pi : -kInv4Pi);
    const int c0 = kq * 2;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = task.row0 + mt * 8 + rq;
      // C/D fragment rows are lane/4 as well, so a lane stores its own row
      bool bad = false;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
        bad = bad || !isfinite(C[mt][nb][0]) || !isfinite(C[mt][nb][1]);
      if (row < task.row0 + task.nrows && bad) verify_row_m(a, task.box, row, DIM);
      if (row >= task.row0 + task.nrows) continue;
      double* u = a.U + (tb.slot + row) * (kNRHS * SW);
      const bool skel_row = row < tb.k;
      double* uh = a.UH + (tb.skel + (skel_row ? row : 0)) * (kNRHS * SW);
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // rhs block c0 + 8*half
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int rhs = c0 + 8 * half + w;
          if (CPLX) {
            u[2 * rhs] = C[mt][half][w] * scale;
            u[2 * rhs + 1] = C[mt][2 + half][w] * scale;
            if (skel_row) {
              uh[2 * rhs] = -H[mt][half][w] * scale;
              uh[2 * rhs + 1] = -H[mt][2 + half][w] * scale;
            }
          } else {
            u[rhs] = C[mt][half][w] * scale;
            if (skel_row) uh[rhs] = -H[mt][half][w] * scale;
          }
        }
      }
    }
  }
}

// ---- tree passes for kNRHS right-hand sides ------------------------------

// K0m: Qm[slot][r] = q[orig + r*N] for r < nc, 0 for the padding columns.
template <class S>
__global__ void k0m_gather(const int64_t* __restrict__ slot, const int32_t* __restrict__ orig,
                           int64_t n_owned, int64_t N, int nc, const S* __restrict__ q,
                           S* __restrict__ Q) {
  const int64_t total = n_owned * kNRHS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kNRHS;
    const int r = (int)(i % kNRHS);
    S v{};
    if (r < nc) v = q[(int64_t)r * N + orig[t]];
    Q[slot[t] * kNRHS + r] = v;
  }
}

template <class S>
__global__ void k4m_scatter(const int64_t* __restrict__ slot, const int32_t* __restrict__ orig,
                            int64_t n_owned, int64_t N, int nc, const S* __restrict__ U,
                            S* __restrict__ u) {
  const int64_t total = n_owned * kNRHS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kNRHS;
    const int r = (int)(i % kNRHS);
    if (r < nc) u[(int64_t)r * N + orig[t]] = U[slot[t] * kNRHS + r];
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 t, double2 u) {  // conj(t) * u
  return make_double2(fma(t.x, u.x, t.y * u.y), fma(t.x, u.y, -t.y * u.x));
}
__device__ __forceinline__ double mulr(double a, double b) { return a * b; }

// K1m: qhat[i][r] = Q[i][r] + sum_j T[i,j] Q[k+j][r]; one CTA per (box, 8 rows),
// thread (row, rhs); q_R streamed through shared memory in chunks of 64.
template <class S>
__global__ void __launch_bounds__(kUpRows * kNRHS) k1m_upward(const LevelItem* __restrict__ items,
                                                  const BoxRec* __restrict__ box,
                                                  const int64_t* __restrict__ T_off,
                                                  const S* __restrict__ T, S* __restrict__ Q,
                                                  S* __restrict__ QH,
                                                  const int64_t* __restrict__ up_dst) {
  __shared__ S sq[64][kNRHS];
  const LevelItem it = items[blockIdx.x];
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  const int li = threadIdx.x / kNRHS, rhs = threadIdx.x % kNRHS;  // kUpRows rows x 16 rhs
  const int i = it.first + li;
  const S* Tb = T + T_off[it.box] + (int64_t)(i < k ? i : 0) * r;
  S acc{};
  for (int j0 = 0; j0 < r; j0 += 64) {
    __syncthreads();
    for (int v = threadIdx.x; v < 64 * kNRHS; v += blockDim.x) {
      const int jj = v / kNRHS, rr = v % kNRHS;
      sq[jj][rr] = j0 + jj < r ? Q[(br.slot + k + j0 + jj) * kNRHS + rr] : S{};
    }
    __syncthreads();
    if (i < k) {
      const int jn = min(64, r - j0);
      for (int jj = 0; jj < jn; ++jj) {
        const S t = Tb[j0 + jj];
        if constexpr (sizeof(S) == 16) {
          const double2 p = cmul(t, sq[jj][rhs]);
          acc.x += p.x;
          acc.y += p.y;
        } else {
          acc = fma(t, sq[jj][rhs], acc);
        }
      }
    }
  }
  if (i < k && i < it.first + kUpRows) {
    S v = Q[(br.slot + i) * kNRHS + rhs];
    if constexpr (sizeof(S) == 16) {
      v.x += acc.x;
      v.y += acc.y;
    } else {
      v += acc;
    }
    QH[(br.skel + i) * kNRHS + rhs] = v;
    Q[up_dst[br.skel + i] * kNRHS + rhs] = v;
  }
}

// K3m: uhat = UH + U[parent]; U_S += uhat; U_R[j][r] += sum_i conj(T[i,j]) uhat[i][r].
// One CTA per (box, 16 columns), thread (column, rhs).
template <class S>
__global__ void __launch_bounds__(256) k3m_downward(const LevelItem* __restrict__ items,
                                                    const BoxRec* __restrict__ box,
                                                    const int64_t* __restrict__ T_off,
                                                    const S* __restrict__ T, S* __restrict__ U,
                                                    const S* __restrict__ UH,
                                                    const int64_t* __restrict__ up_dst) {
  extern __shared__ unsigned char smraw[];
  S* su = reinterpret_cast<S*>(smraw);  // [k][kNRHS]
  const LevelItem it = items[blockIdx.x];
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  for (int v = threadIdx.x; v < k * kNRHS; v += blockDim.x) {
    const int i = v / kNRHS, rr = v % kNRHS;
    S a = UH[(br.skel + i) * kNRHS + rr], b = U[up_dst[br.skel + i] * kNRHS + rr];
    S s;
    if constexpr (sizeof(S) == 16) {
      s = make_double2(a.x + b.x, a.y + b.y);
    } else {
      s = a + b;
    }
    su[v] = s;
    if (it.first == 0) {
      S o = U[(br.slot + i) * kNRHS + rr];
      if constexpr (sizeof(S) == 16) {
        U[(br.slot + i) * kNRHS + rr] = make_double2(o.x + s.x, o.y + s.y);
      } else {
        U[(br.slot + i) * kNRHS + rr] = o + s;
      }
    }
  }
  __syncthreads();
  const int jl = threadIdx.x / kNRHS, rhs = threadIdx.x % kNRHS;
  const int j = it.first + jl;
  if (j >= r) return;
  const S* Tb = T + T_off[it.box] + j;
  S acc{};
  for (int i = 0; i < k; ++i) {
    const S t = Tb[(int64_t)i * r];
    if constexpr (sizeof(S) == 16) {
      const double2 p = cmulc(t, su[i * kNRHS + rhs]);
      acc.x += p.x;
      acc.y += p.y;
    } else {
      acc = fma(t, su[i * kNRHS + rhs], acc);
    }
  }
  S o = U[(br.slot + k + j) * kNRHS + rhs];
  if constexpr (sizeof(S) == 16) {
    U[(br.slot + k + j) * kNRHS + rhs] = make_double2(o.x + acc.x, o.y + acc.y);
  } else {
    U[(br.slot + k + j) * kNRHS + rhs] = o + acc;
  }
}

int grid_m(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

}  // namespace

int configure_multi(DevPlan& p, int device, size_t max_k) {
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  cudaError_t e;
  if (p.kernel == SFMM_HELMHOLTZ3D)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2m_translate<SFMM_HELMHOLTZ3D>, kMThreads, 0);
  else if (p.kernel == SFMM_LAPLACE3D)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2m_translate<SFMM_LAPLACE3D>, kMThreads, 0);
  else
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2m_translate<SFMM_LAPLACE2D>, kMThreads, 0);
  if (e != cudaSuccess) return -1;
  p.k2m_grid = sms * std::max(1, per_sm);
  const size_t sw = p.cplx ? 16 : 8;
  p.down_m_smem = std::max<size_t>(max_k * kNRHS * sw, 16);
  if (p.down_m_smem > 48 * 1024) {
    const void* f = p.cplx ? (const void*)k3m_downward<double2> : (const void*)k3m_downward<double>;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.down_m_smem) !=
        cudaSuccess)
      return -1;
  }
  return 0;
}

void launch_gather_m(const DevPlan& p, const double* q, int nc, DevState& s, cudaStream_t st) {
  const int g = grid_m(p.n_owned_points * kNRHS);
  if (p.cplx)
    k0m_gather<double2><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.n_owned_points, p.n_points, nc,
                                           reinterpret_cast<const double2*>(q),
                                           reinterpret_cast<double2*>(s.Q));
  else
    k0m_gather<double><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.n_owned_points, p.n_points, nc,
                                          q, s.Q);
}

void launch_scatter_m(const DevPlan& p, const DevState& s, double* u, int nc, cudaStream_t st) {
  const int g = grid_m(p.n_owned_points * kNRHS);
  if (p.cplx)
    k4m_scatter<double2><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.n_owned_points, p.n_points, nc,
                                            reinterpret_cast<const double2*>(s.U),
                                            reinterpret_cast<double2*>(u));
  else
    k4m_scatter<double><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.n_owned_points, p.n_points, nc,
                                           s.U, u);
}

void launch_upward_m(const DevPlan& p, const HostPlan& hp, int level, DevState& s, cudaStream_t st) {
  const int64_t i0 = hp.up_lvl[level], i1 = hp.up_lvl[level + 1];
  if (i1 <= i0) return;
  if (p.cplx)
    k1m_upward<double2><<<(unsigned)(i1 - i0), kUpRows * kNRHS, 0, st>>>(
        p.up_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.Q), reinterpret_cast<double2*>(s.QH), p.up_dst);
  else
    k1m_upward<double><<<(unsigned)(i1 - i0), kUpRows * kNRHS, 0, st>>>(p.up_items + i0, p.box, p.T_off, p.T,
                                                             s.Q, s.QH, p.up_dst);
}

void launch_downward_m(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                       cudaStream_t st) {
  const int64_t i0 = hp.down_m_lvl[level], i1 = hp.down_m_lvl[level + 1];
  if (i1 <= i0) return;
  if (p.cplx)
    k3m_downward<double2><<<(unsigned)(i1 - i0), 256, p.down_m_smem, st>>>(
        p.down_m_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.U), reinterpret_cast<const double2*>(s.UH), p.up_dst);
  else
    k3m_downward<double><<<(unsigned)(i1 - i0), 256, p.down_m_smem, st>>>(
        p.down_m_items + i0, p.box, p.T_off, p.T, s.U, s.UH, p.up_dst);
}

void launch_translate_m(const DevPlan& p, DevState& s, cudaStream_t st) {
  const size_t sw = p.cplx ? 16 : 8;
  cudaMemsetAsync(s.U, 0, (size_t)p.n_slots * kNRHS * sw, st);
  cudaMemsetAsync(s.UH, 0, (size_t)p.n_skel * kNRHS * sw, st);
  if (p.n_tasks_m == 0) return;
  K2MArgs a;
  a.box = p.box;
  a.er = p.ent_range_full;
  a.ent = p.entries_full;
  a.tasks = p.tasks_m;
  a.n_tasks = p.n_tasks_m;
  a.X = p.X;
  a.Y = p.Y;
  a.Z = p.Z;
  a.sid = p.slot_id;
  a.Q = s.Q;
  a.QH = s.QH;
  a.U = s.U;
  a.UH = s.UH;
  a.counter = p.counter + 2;
  a.err = p.err_flag;
  a.kappa = p.kappa;
  cudaMemsetAsync(p.counter + 2, 0, sizeof(int), st);
  const int grid = (int)std::min<int64_t>(p.k2m_grid, (p.n_tasks_m + kMWarps - 1) / kMWarps);
  if (p.kernel == SFMM_HELMHOLTZ3D)
    k2m_translate<SFMM_HELMHOLTZ3D><<<grid, kMThreads, 0, st>>>(a);
  else if (p.kernel == SFMM_LAPLACE3D)
    k2m_translate<SFMM_LAPLACE3D><<<grid, kMThreads, 0, st>>>(a);
  else
    k2m_translate<SFMM_LAPLACE2D><<<grid, kMThreads, 0, st>>>(a);
}

}  // namespace sfmm_gpu
