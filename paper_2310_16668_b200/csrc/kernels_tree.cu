// K0/K1/K3/K4/K5: leaf gather, interpolation GEMVs, leaf scatter and the
// dense fallback of the sm_100a SRS-FMM apply.
//
//   K0 gather   <- upward_pass leaf branch   apply.cpp:124-125
//   K1 upward   <- upward_pass l >= 2        apply.cpp:126-143
//   K3 downward <- downward_pass             apply.cpp:274-293
//   K4 scatter  <- downward_pass leaf loop   apply.cpp:294-302
//   K5 direct   <- fmm_apply depth < 2       apply.cpp:316-328, oracle.cpp:9-49
//
// K1 and K3 read every interpolation matrix T exactly once per apply with
// coalesced row (K1) or column (K3) sweeps; they are HBM-bound.  Slots of a
// compressed box are stored [skeleton | redundant], so the vectors they touch
// are contiguous.
#include <algorithm>
#include <cstdlib>

#include "launch.h"

namespace sfmm_gpu {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kUpThreads = 256;
constexpr double kInv4Pi = 0.0795774715459476678844418816862571810;

// K0 + the leaf-level K1 copy: Q[slot] = q[orig]; for a point of an
// uncompressed leaf (k = n: every slot is a skeleton slot) also qhat = q and
// the parent's slot (k1_copy's work, apply.cpp:124-131, fused here so the
// leaf charges are read once).  int32 maps: 12 B of indices per point.
template <class S>
__device__ __forceinline__ void k0_point(int64_t t, const int32_t* __restrict__ slot,
                                         const int32_t* __restrict__ orig,
                                         const int32_t* __restrict__ hat,
                                         const int32_t* __restrict__ up_dst,
                                         const S* __restrict__ q, S* __restrict__ Q,
                                         S* __restrict__ QH) {
  const S v = __ldg(q + __ldg(orig + t));
  Q[__ldg(slot + t)] = v;
  const int32_t h = __ldg(hat + t);
  if (h >= 0) {
    QH[h] = v;
    Q[__ldg(up_dst + h)] = v;
  }
}

template <class S>
__global__ void __launch_bounds__(256) k0_gather(const int32_t* __restrict__ slot,
                                                 const int32_t* __restrict__ orig,
                                                 const int32_t* __restrict__ hat,
                                                 const int32_t* __restrict__ up_dst, int64_t n,
                                                 const S* __restrict__ q, S* __restrict__ Q,
                                                 S* __restrict__ QH) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    k0_point<S>(t, slot, orig, hat, up_dst, q, Q, QH);
}

// K4 + the leaf-level K3 copy: u[orig] = U[slot] (+ uhat + the parent's
// potential for a point of an uncompressed leaf, apply.cpp:284-301), in the
// order k3_copy adds them, so the result is bit-identical to the unfused pair.
template <class S>
__global__ void __launch_bounds__(256) k4_scatter(const int32_t* __restrict__ slot,
                                                  const int32_t* __restrict__ orig,
                                                  const int32_t* __restrict__ hat,
                                                  const int32_t* __restrict__ up_dst, int64_t n,
                                                  const S* __restrict__ U,
                                                  const S* __restrict__ UH, S* __restrict__ u);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// K1, real: qhat_i = q_S[i] + sum_j T[i,j] q_R[j] for up to kUpRows1 rows of
// one box.  Each warp streams 4 rows of T at once (4 independent coalesced
// loads per lane per step, four steps unrolled: 5.2 vs 4.9 TB/s at two, and
// slower again at eight or with 8 rows per warp); q_R (shared by all rows of
// the box) is staged in shared memory first (measured: 2.9 vs 2.3 TB/s for
// reading it through the read-only cache).
constexpr int kUpRowsPerWarp = 4;
// Q is read through L2 (ld.cg): in the persistent tree pass the charges were
// written by other CTAs of the same launch.
__device__ __forceinline__ void k1_real_item(const LevelItem it, const BoxRec* __restrict__ box,
                                             const int64_t* __restrict__ T_off,
                                             const double* __restrict__ T, double* __restrict__ Q,
                                             double* __restrict__ QH,
                                             const int32_t* __restrict__ up_dst, double* smq) {
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  for (int j = threadIdx.x; j < r; j += blockDim.x) smq[j] = __ldcg(Q + br.slot + k + j);
  __syncthreads();
  const double* qR = smq;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* Tb = T + T_off[it.box];
  const int i1 = min(it.first + kUpRows1, k);
  for (int i0 = it.first + w * kUpRowsPerWarp; i0 < i1; i0 += (kUpThreads / 32) * kUpRowsPerWarp) {
    double acc[kUpRowsPerWarp];
    const double* Ti[kUpRowsPerWarp];
#pragma unroll
    for (int m = 0; m < kUpRowsPerWarp; ++m) {
      acc[m] = 0.0;
      Ti[m] = Tb + (int64_t)min(i0 + m, i1 - 1) * r;
    }
#pragma unroll 4
    for (int j = lane; j < r; j += 32) {
      const double qj = qR[j];
#pragma unroll
      for (int m = 0; m < kUpRowsPerWarp; ++m) acc[m] = fma(__ldg(Ti[m] + j), qj, acc[m]);
    }
#pragma unroll
    for (int m = 0; m < kUpRowsPerWarp; ++m) {
      const double s = warp_sum(acc[m]);
      const int i = i0 + m;
      if (lane == 0 && i < i1) {
        const double v = __ldcg(Q + br.slot + i) + s;
        QH[br.skel + i] = v;
        Q[up_dst[br.skel + i]] = v;
      }
    }
  }
}

__global__ void __launch_bounds__(kUpThreads) k1_upward_real(
    const LevelItem* __restrict__ items, const BoxRec* __restrict__ box,
    const int64_t* __restrict__ T_off, const double* __restrict__ T, double* __restrict__ Q,
    double* __restrict__ QH, const int32_t* __restrict__ up_dst) {
  extern __shared__ double smq[];
  k1_real_item(items[blockIdx.x], box, T_off, T, Q, QH, up_dst, smq);
}

// K1, real, with the T rows staged by the bulk-copy engine (TMA, cp.async.bulk
// -> SASS UBLKCP) instead of register loads: the CTA's 64-row slice of T is
// contiguous (row-major k x r per box), so it moves as a few large copies into
// a 3-deep ring of shared-memory stages, each completing on an mbarrier; the
// eight warps reduce rows from shared memory.  Up to 3 x 32 KB are in flight
// per CTA (two CTAs per SM) with no registers held for them -- the HBM
// stream K1 is bound by (8 B per T entry).
constexpr int kK1Stages = 4;
constexpr int kK1StageBytes = 32 * 1024;
constexpr int kK1MaxR = (kK1StageBytes - 16) / 8;  // longest row one stage holds

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Persistent and warp-specialized: CTA g takes items g, g + grid, ...; each
// item (box, 64-row slice) is cut into jobs of up to rows_ps rows whose T rows
// (contiguous) and the box's q_R arrive together in one ring stage.  A
// producer warp (one lane) walks the job list, waits for a stage to be freed
// (`empty` mbarrier, one arrival per consumer warp), publishes the job's
// geometry in shared memory and issues the bulk copies onto the stage's
// `full` mbarrier; eight consumer warps wait on `full`, reduce the rows from
// shared memory and free the stage.  The producer's metadata loads overlap
// the consumers' work, so the copy engine always has kK1Stages jobs queued.
struct K1Meta {
  int row0, nr, r, qo, to;  // first row, rows, row length, q_R / T offsets in the stage
  int pad;
  int64_t slot, skel;
};
constexpr int kK1Consumers = kUpThreads / 32;        // 8 consumer warps
constexpr int kK1BulkThreads = kUpThreads + 32;       // + 1 producer warp

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kK1BulkThreads, 1) k1_upward_real_bulk(
    const LevelItem* __restrict__ items, int64_t n_items, const BoxRec* __restrict__ box,
    const int64_t* __restrict__ T_off, const double* __restrict__ T, double* __restrict__ Q,
    double* __restrict__ QH, const int32_t* __restrict__ up_dst, int qr_cap) {
  extern __shared__ __align__(128) unsigned char k1sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(k1sm);
  uint64_t* empty = full + kK1Stages;
  K1Meta* meta = reinterpret_cast<K1Meta*>(k1sm + 128);
  double* ring = reinterpret_cast<double*>(k1sm + 128 + 64 * kK1Stages);
  const int stage_d = qr_cap + kK1StageBytes / 8;  // doubles per stage: [q_R | T rows]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kK1Stages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kK1Consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kK1Consumers) {  // ---- producer ----
    if (lane != 0) return;
    int job = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const LevelItem it = items[item];
      const BoxRec br = box[it.box];
      const int r = br.n - br.k;
      const int i0 = it.first, i1 = min(it.first + kUpRows1, br.k);
      const int rows_ps = max(1, min(i1 - i0, kK1MaxR / r));
      const double* qs = Q + br.slot + br.k;
      const int oq = (int)((reinterpret_cast<uintptr_t>(qs) >> 3) & 1);
      const uint32_t bq = (uint32_t)(((oq + r) * 8 + 15) & ~15);
      const double* tb = T + T_off[it.box];
      for (int row0 = i0; row0 < i1; row0 += rows_ps, ++job) {
        const int st = job % kK1Stages;
        if (job >= kK1Stages) mbar_wait(&empty[st], (uint32_t)(((job / kK1Stages) - 1) & 1));
        const int nr = min(rows_ps, i1 - row0);
        const double* ts = tb + (int64_t)row0 * r;
        const int ot = (int)((reinterpret_cast<uintptr_t>(ts) >> 3) & 1);
        const uint32_t bt = (uint32_t)(((ot + nr * r) * 8 + 15) & ~15);
        meta[st] = K1Meta{row0, nr, r, oq, qr_cap + ot, 0, br.slot, br.skel};
        double* dst = ring + (int64_t)st * stage_d;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], bq + bt);
        bulk_g2s(dst, qs - oq, bq, &full[st]);
        bulk_g2s(dst + qr_cap, ts - ot, bt, &full[st]);
      }
    }
    // end marker: an empty job (nr = 0) released by a plain arrive
    const int st = job % kK1Stages;
    if (job >= kK1Stages) mbar_wait(&empty[st], (uint32_t)(((job / kK1Stages) - 1) & 1));
    meta[st].nr = 0;
    mbar_arrive(&full[st]);
    return;
  }
  // ---- consumers ----
  for (int job = 0;; ++job) {
    const int st = job % kK1Stages;
    mbar_wait(&full[st], (uint32_t)((job / kK1Stages) & 1));
    const K1Meta m = meta[st];
    if (m.nr == 0) break;
    const double* stg = ring + (int64_t)st * stage_d;
    const double* qR = stg + m.qo;
    const double* Ts = stg + m.to;
    const int r = m.r;
    for (int m0 = warp * kUpRowsPerWarp; m0 < m.nr; m0 += kK1Consumers * kUpRowsPerWarp) {
      double acc[kUpRowsPerWarp];
#pragma unroll
      for (int u = 0; u < kUpRowsPerWarp; ++u) acc[u] = 0.0;
      for (int j = lane; j < r; j += 32) {
        const double qj = qR[j];
#pragma unroll
        for (int u = 0; u < kUpRowsPerWarp; ++u)
          acc[u] = fma(Ts[min(m0 + u, m.nr - 1) * r + j], qj, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < kUpRowsPerWarp; ++u) {
        const double sum = warp_sum(acc[u]);
        if (lane == 0 && m0 + u < m.nr) {
          const int i = m.row0 + m0 + u;
          const double v = Q[m.slot + i] + sum;
          QH[m.skel + i] = v;
          Q[up_dst[m.skel + i]] = v;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// K1, complex.
__device__ __forceinline__ void k1_cplx_item(const LevelItem it, const BoxRec* __restrict__ box,
                                             const int64_t* __restrict__ T_off,
                                             const double2* __restrict__ T,
                                             double2* __restrict__ Q, double2* __restrict__ QH,
                                             const int32_t* __restrict__ up_dst, double2* smq2) {
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  for (int j = threadIdx.x; j < r; j += blockDim.x) smq2[j] = __ldcg(Q + br.slot + k + j);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* Tb = T + T_off[it.box];
  const int i1 = min(it.first + kUpRows1, k);
  for (int i = it.first + w; i < i1; i += kUpThreads / 32) {
    const double2* Ti = Tb + (int64_t)i * r;
    double ar = 0.0, ai = 0.0;
    for (int j = lane; j < r; j += 32) {
      const double2 t = __ldg(Ti + j), x = smq2[j];
      ar = fma(t.x, x.x, fma(-t.y, x.y, ar));
      ai = fma(t.x, x.y, fma(t.y, x.x, ai));
    }
    ar = warp_sum(ar);
    ai = warp_sum(ai);
    if (lane == 0) {
      const double2 q = __ldcg(Q + br.slot + i);
      const double2 v = make_double2(q.x + ar, q.y + ai);
      QH[br.skel + i] = v;
      Q[up_dst[br.skel + i]] = v;
    }
  }
}

__global__ void __launch_bounds__(kUpThreads) k1_upward_cplx(
    const LevelItem* __restrict__ items, const BoxRec* __restrict__ box,
    const int64_t* __restrict__ T_off, const double2* __restrict__ T, double2* __restrict__ Q,
    double2* __restrict__ QH, const int32_t* __restrict__ up_dst) {
  extern __shared__ double2 smq2[];
  k1_cplx_item(items[blockIdx.x], box, T_off, T, Q, QH, up_dst, smq2);
}

// K1 / K3 for uncompressed boxes (k = n, r = 0: no interpolation block), one
// warp per box: qhat = q (K1) and U_S += UH + U[parent slice] (K3).
__device__ __forceinline__ double add_s(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add_s(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}

template <class S>
__device__ __forceinline__ void k4_point(int64_t t, const int32_t* __restrict__ slot,
                                         const int32_t* __restrict__ orig,
                                         const int32_t* __restrict__ hat,
                                         const int32_t* __restrict__ up_dst,
                                         const S* __restrict__ U, const S* __restrict__ UH,
                                         S* __restrict__ u) {
  S v = __ldcg(U + __ldg(slot + t));
  const int32_t h = __ldg(hat + t);
  if (h >= 0) v = add_s(v, add_s(__ldcg(UH + h), __ldcg(U + __ldg(up_dst + h))));
  u[__ldg(orig + t)] = v;
}

template <class S>
__global__ void __launch_bounds__(256) k4_scatter(const int32_t* __restrict__ slot,
                                                  const int32_t* __restrict__ orig,
                                                  const int32_t* __restrict__ hat,
                                                  const int32_t* __restrict__ up_dst, int64_t n,
                                                  const S* __restrict__ U,
                                                  const S* __restrict__ UH, S* __restrict__ u) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    k4_point<S>(t, slot, orig, hat, up_dst, U, UH, u);
}

// K4 in two coalesced-write passes (single-rank plans: every point owned):
// k4_fold writes each owned point's potential in slot order (same arithmetic
// as k4_point), k4_gather reads it back in the ORIGINAL order through the
// inverse map, so the random side is a read (the fold's output still sits in
// L2) instead of a partial-sector write.
template <class S>
__global__ void __launch_bounds__(256) k4_fold(const int32_t* __restrict__ slot,
                                               const int32_t* __restrict__ hat,
                                               const int32_t* __restrict__ up_dst, int64_t n,
                                               const S* __restrict__ U, const S* __restrict__ UH,
                                               S* __restrict__ V) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    S v = __ldcg(U + __ldg(slot + t));
    const int32_t h = __ldg(hat + t);
    if (h >= 0) v = add_s(v, add_s(__ldcg(UH + h), __ldcg(U + __ldg(up_dst + h))));
    V[t] = v;
  }
}

template <class S>
__global__ void __launch_bounds__(256) k4_gather(const int32_t* __restrict__ pos, int64_t n,
                                                 const S* __restrict__ V, S* __restrict__ u) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    u[i] = __ldcg(V + __ldg(pos + i));
}

__global__ void k_invert_orig(const int32_t* __restrict__ orig, int64_t n, int32_t* __restrict__ pos) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    pos[orig[t]] = (int32_t)t;
}

__device__ __forceinline__ double shfl_s(double v, int src) { return __shfl_sync(kFull, v, src); }
__device__ __forceinline__ double2 shfl_s(double2 v, int src) {
  return make_double2(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src));
}
__device__ __forceinline__ double fma_s(double t, double q, double acc) { return fma(t, q, acc); }
__device__ __forceinline__ double2 fma_s(double2 t, double2 q, double2 acc) {  // acc + t q
  return make_double2(fma(t.x, q.x, fma(-t.y, q.y, acc.x)), fma(t.x, q.y, fma(t.y, q.x, acc.y)));
}
__device__ __forceinline__ double fma_cs(double t, double u, double acc) { return fma(t, u, acc); }
__device__ __forceinline__ double2 fma_cs(double2 t, double2 u, double2 acc) {  // acc + conj(t) u
  return make_double2(fma(t.x, u.x, fma(t.y, u.y, acc.x)), fma(t.x, u.y, fma(-t.y, u.x, acc.y)));
}

// One box per warp (uncompressed boxes, r = 0: copies only; boxes with a
// short interpolation block, 0 < r <= kWarpBoxR: lane = row of T, q_R held
// one entry per lane and broadcast by shuffles -- no reduction, no idle CTA
// threads, on adaptive trees most boxes of the deepest levels).
template <class S>
__device__ __forceinline__ void k1_copy_box(const BoxRec br, int lane, const S* __restrict__ Tb,
                                            S* __restrict__ Q, S* __restrict__ QH,
                                            const int32_t* __restrict__ up_dst) {
  const int k = br.k, r = br.n - br.k;
  const S qr = lane < r ? __ldcg(Q + br.slot + k + lane) : S{};
  for (int i0 = 0; i0 < k; i0 += 32) {
    const int i = i0 + lane;
    S acc{};
    for (int j = 0; j < r; ++j) {
      const S q = shfl_s(qr, j);
      if (i < k) acc = fma_s(Tb[(int64_t)i * r + j], q, acc);
    }
    if (i < k) {
      const S q = __ldcg(Q + br.slot + i);
      const S v = r > 0 ? add_s(q, acc) : q;
      QH[br.skel + i] = v;
      Q[up_dst[br.skel + i]] = v;
    }
  }
}

template <class S>
__device__ __forceinline__ void k3_copy_box(const BoxRec br, int lane, const S* __restrict__ Tb,
                                            S* __restrict__ U, const S* __restrict__ UH,
                                            const int32_t* __restrict__ up_dst) {
  const int k = br.k, r = br.n - br.k;
  S acc{};  // lane j < r: U_R[j] += sum_i conj(T[i,j]) uhat[i]
  for (int i0 = 0; i0 < k; i0 += 32) {
    const int i = i0 + lane;
    S uh{};
    if (i < k) {
      uh = add_s(__ldcg(UH + br.skel + i), __ldcg(U + up_dst[br.skel + i]));
      U[br.slot + i] = add_s(__ldcg(U + br.slot + i), uh);
    }
    const int cnt = min(32, k - i0);
    for (int ii = 0; ii < cnt && r > 0; ++ii) {
      const S u = shfl_s(uh, ii);
      if (lane < r) acc = fma_cs(Tb[(int64_t)(i0 + ii) * r + lane], u, acc);
    }
  }
  if (lane < r) U[br.slot + k + lane] = add_s(__ldcg(U + br.slot + k + lane), acc);
}

template <class S>
__global__ void __launch_bounds__(256) k1_copy(const int32_t* __restrict__ boxes, int64_t nbox,
                                               const BoxRec* __restrict__ box,
                                               const int64_t* __restrict__ T_off,
                                               const S* __restrict__ T, S* __restrict__ Q,
                                               S* __restrict__ QH, const int32_t* __restrict__ up_dst) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nbox) return;
  const int32_t b = boxes[w];
  k1_copy_box<S>(box[b], threadIdx.x & 31, T + T_off[b], Q, QH, up_dst);
}

template <class S>
__global__ void __launch_bounds__(256) k3_copy(const int32_t* __restrict__ boxes, int64_t nbox,
                                               const BoxRec* __restrict__ box,
                                               const int64_t* __restrict__ T_off,
                                               const S* __restrict__ T, S* __restrict__ U,
                                               const S* __restrict__ UH,
                                               const int32_t* __restrict__ up_dst) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nbox) return;
  const int32_t b = boxes[w];
  k3_copy_box<S>(box[b], threadIdx.x & 31, T + T_off[b], U, UH, up_dst);
}

// K3, real: uhat = UH + U[parent slice]; U_S += uhat; U_R += T^T uhat.
// U is read through L2 (ld.cg): in the persistent tree pass the parent's
// potentials were written by other CTAs of the same launch.
__device__ __forceinline__ void k3_real_item(const LevelItem it, const BoxRec* __restrict__ box,
                                             const int64_t* __restrict__ T_off,
                                             const double* __restrict__ T, double* __restrict__ U,
                                             const double* __restrict__ UH,
                                             const int32_t* __restrict__ up_dst, double* smu) {
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double v = __ldcg(UH + br.skel + i) + __ldcg(U + up_dst[br.skel + i]);
    smu[i] = v;
    if (it.first == 0) U[br.slot + i] = __ldcg(U + br.slot + i) + v;
  }
  __syncthreads();
  const int j = it.first + threadIdx.x;
  if (j >= r) return;
  const double* Tb = T + T_off[it.box] + j;
  double acc = 0.0;
#pragma unroll 4
  for (int i = 0; i < k; ++i) acc = fma(Tb[(int64_t)i * r], smu[i], acc);
  U[br.slot + k + j] = __ldcg(U + br.slot + k + j) + acc;
}

__global__ void __launch_bounds__(kDownCols) k3_downward_real(
    const LevelItem* __restrict__ items, const BoxRec* __restrict__ box,
    const int64_t* __restrict__ T_off, const double* __restrict__ T, double* __restrict__ U,
    const double* __restrict__ UH, const int32_t* __restrict__ up_dst) {
  extern __shared__ double smu[];
  k3_real_item(items[blockIdx.x], box, T_off, T, U, UH, up_dst, smu);
}

// K3, complex: U_R += conj(T)^T uhat (apply.cpp:290).
__device__ __forceinline__ void k3_cplx_item(const LevelItem it, const BoxRec* __restrict__ box,
                                             const int64_t* __restrict__ T_off,
                                             const double2* __restrict__ T,
                                             double2* __restrict__ U, const double2* __restrict__ UH,
                                             const int32_t* __restrict__ up_dst, double2* smu2) {
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double2 a = __ldcg(UH + br.skel + i), b = __ldcg(U + up_dst[br.skel + i]);
    const double2 v = make_double2(a.x + b.x, a.y + b.y);
    smu2[i] = v;
    if (it.first == 0) {
      double2 o = __ldcg(U + br.slot + i);
      U[br.slot + i] = make_double2(o.x + v.x, o.y + v.y);
    }
  }
  __syncthreads();
  const int j = it.first + threadIdx.x;
  if (j >= r) return;
  const double2* Tb = T + T_off[it.box] + j;
  double ar = 0.0, ai = 0.0;
#pragma unroll 4
  for (int i = 0; i < k; ++i) {
    const double2 t = Tb[(int64_t)i * r], u = smu2[i];
    ar = fma(t.x, u.x, fma(t.y, u.y, ar));
    ai = fma(t.x, u.y, fma(-t.y, u.x, ai));
  }
  double2 o = __ldcg(U + br.slot + k + j);
  U[br.slot + k + j] = make_double2(o.x + ar, o.y + ai);
}

__global__ void __launch_bounds__(kDownCols) k3_downward_cplx(
    const LevelItem* __restrict__ items, const BoxRec* __restrict__ box,
    const int64_t* __restrict__ T_off, const double2* __restrict__ T, double2* __restrict__ U,
    const double2* __restrict__ UH, const int32_t* __restrict__ up_dst) {
  extern __shared__ double2 smu2[];
  k3_cplx_item(items[blockIdx.x], box, T_off, T, U, UH, up_dst, smu2);
}

// Kernel value exactly as the reference writes it (kernel.hpp:40-71), with
// every operation rounded separately (no FMA contraction), so the depth < 2
// fallback reproduces direct_sum's arithmetic.
__device__ __forceinline__ double2 ref_from_r2(int kernel, double kappa, double r2) {
  const double pi4 = 4.0 * 3.14159265358979323846264338327950288;
  if (kernel == SFMM_LAPLACE3D) return make_double2(__ddiv_rn(1.0, __dmul_rn(pi4, __dsqrt_rn(r2))), 0.0);
  if (kernel == SFMM_LAPLACE2D) return make_double2(__dmul_rn(log(r2), -1.0 / pi4), 0.0);
  const double r = __dsqrt_rn(r2);
  const double kr = __dmul_rn(kappa, r);
  const double r4 = __dmul_rn(4.0, r);
  return make_double2(__ddiv_rn(cos(kr), r4), __ddiv_rn(sin(kr), r4));
}

__device__ __forceinline__ double ref_r2(const double* xi, const double* xj, int dim) {
  double r2 = 0.0;
  for (int k = 0; k < dim; ++k) {
    const double dx = __dsub_rn(xi[k], xj[k]);
    r2 = __dadd_rn(r2, __dmul_rn(dx, dx));
  }
  return r2;
}

// K5: one thread per target, sources ascending, j == i skipped (oracle.cpp:9-31).
__global__ void k5_direct(int kernel, double kappa, int dim, int cplx, int64_t n,
                          const double* __restrict__ pts, const double* __restrict__ q,
                          double* __restrict__ u, int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xi[3];
  for (int k = 0; k < dim; ++k) xi[k] = pts[i * dim + k];
  double ar = 0.0, ai = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue;
    const double r2 = ref_r2(xi, pts + j * dim, dim);
    if (r2 == 0.0) {
      atomicOr(err, 1);
      continue;
    }
    const double2 g = ref_from_r2(kernel, kappa, r2);
    if (cplx) {
      const double qr = q[2 * j], qi = q[2 * j + 1];
      ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(g.x, qr), __dmul_rn(g.y, qi)));
      ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(g.x, qi), __dmul_rn(g.y, qr)));
    } else {
      ar = __dadd_rn(ar, __dmul_rn(g.x, q[j]));
    }
  }
  if (cplx) {
    u[2 * i] = ar;
    u[2 * i + 1] = ai;
  } else {
    u[i] = ar;
  }
}

// Dense subset sum for accuracy checks: one CTA per target, block reduction.
__global__ void __launch_bounds__(256) k5_direct_subset(int kernel, double kappa, int dim,
                                                        int cplx, int64_t n,
                                                        const double* __restrict__ pts,
                                                        const double* __restrict__ q,
                                                        const int32_t* __restrict__ targets,
                                                        double* __restrict__ u, int* err) {
  __shared__ double red[2][8];
  const int64_t i = targets[blockIdx.x];
  double xi[3];
  for (int k = 0; k < dim; ++k) xi[k] = pts[i * dim + k];
  double ar = 0.0, ai = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    if (j == i) continue;
    const double r2 = ref_r2(xi, pts + j * dim, dim);
    if (r2 == 0.0) {
      atomicOr(err, 1);
      continue;
    }
    const double2 g = ref_from_r2(kernel, kappa, r2);
    if (cplx) {
      const double qr = q[2 * j], qi = q[2 * j + 1];
      ar += g.x * qr - g.y * qi;
      ai += g.x * qi + g.y * qr;
    } else {
      ar += g.x * q[j];
    }
  }
  ar = warp_sum(ar);
  ai = warp_sum(ai);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][w] = ar;
    red[1][w] = ai;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sr = 0, si = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      sr += red[0][k];
      si += red[1][k];
    }
    if (cplx) {
      u[2 * blockIdx.x] = sr;
      u[2 * blockIdx.x + 1] = si;
    } else {
      u[blockIdx.x] = sr;
    }
  }
}

// Device-side plan build, one warp per box: slot
// geometry and ids (make_plan's gathered coordinates, apply.cpp:70-107) and
// the upward destinations (skeleton.cpp:204-218; apply.cpp:127-131).
__global__ void k_build_slots(SlotBuildArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.n_boxes) return;
  const BoxRec br = a.box[w];
  if (br.slot < 0) return;  // not on this rank (compact slot space of a sharded plan)
  for (int32_t p = lane; p < br.n; p += 32) {
    const int64_t e = br.slot + p;
    const int64_t s = br.slot + a.posmap[e];
    const int64_t id = a.iv[e];
    a.slot_id[s] = (int32_t)id;
    a.X[s] = a.pts[id * a.dim];
    a.Y[s] = a.pts[id * a.dim + 1];
    a.Z[s] = a.dim == 3 ? a.pts[id * a.dim + 2] : 0.0;
  }
  if (br.k > 0 && a.box[a.parent[w]].slot >= 0) {  // (a ghost box's parent may be absent)
    const int64_t ps = a.box[a.parent[w]].slot;
    const int64_t off = a.parent_offset[w];
    for (int32_t i = lane; i < br.k; i += 32)
      a.up_dst[br.skel + i] = (int32_t)(ps + a.posmap[ps + off + i]);
  }
}

// Leaf gather/scatter maps, one warp per owned leaf: index_vec position p of
// the leaf (tree-order point begin + p, original index perm[begin + p]) owns
// slot s0 + posmap[p]; entries are written in slot order.
__global__ void k_build_leaf_maps(SlotBuildArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.n_leaves) return;
  const BoxRec br = a.box[a.leaf_box[w]];
  const int64_t out = a.leaf_out[w], begin = a.leaf_begin[w];
  const bool copy = a.leaf_copy[w] != 0;
  for (int32_t p = lane; p < br.n; p += 32) {
    const int32_t j = a.posmap[br.slot + p];
    a.leaf_slot[out + j] = (int32_t)(br.slot + j);
    a.leaf_orig[out + j] = a.perm[begin + p];
    a.leaf_hat[out + j] = copy ? (int32_t)(br.skel + j) : -1;
  }
}

// One tree level in ONE launch: blocks [0, n_copy_blocks) do the level's
// uncompressed boxes' copies (8 boxes per block, warp per box), the rest its
// interpolation items (K1 upward / K3 downward), so each level costs one
// launch instead of two (launch-bound small plans).
template <class S, bool UP>
__global__ void __launch_bounds__(kUpThreads) k_level(const int32_t* __restrict__ copy_boxes,
                                                     int64_t n_copy, int n_copy_blocks,
                                                     const LevelItem* __restrict__ items,
                                                     const BoxRec* __restrict__ box,
                                                     const int64_t* __restrict__ T_off,
                                                     const double* __restrict__ T,
                                                     double* __restrict__ V, double* __restrict__ VH,
                                                     const int32_t* __restrict__ up_dst) {
  static_assert(kUpThreads == kDownCols, "one block shape for K1 and K3 items");
  extern __shared__ __align__(16) unsigned char lv_smem[];
  if ((int)blockIdx.x < n_copy_blocks) {
    const int64_t w = (int64_t)blockIdx.x * (kUpThreads / 32) + (threadIdx.x >> 5);
    if (w >= n_copy) return;
    const int32_t b = copy_boxes[w];
    const S* Tb = reinterpret_cast<const S*>(T) + T_off[b];
    if (UP)
      k1_copy_box<S>(box[b], threadIdx.x & 31, Tb, reinterpret_cast<S*>(V), reinterpret_cast<S*>(VH),
                     up_dst);
    else
      k3_copy_box<S>(box[b], threadIdx.x & 31, Tb, reinterpret_cast<S*>(V),
                     reinterpret_cast<const S*>(VH), up_dst);
    return;
  }
  const LevelItem it = items[blockIdx.x - n_copy_blocks];
  if constexpr (sizeof(S) == 16) {
    if (UP)
      k1_cplx_item(it, box, T_off, reinterpret_cast<const double2*>(T), reinterpret_cast<double2*>(V),
                   reinterpret_cast<double2*>(VH), up_dst, reinterpret_cast<double2*>(lv_smem));
    else
      k3_cplx_item(it, box, T_off, reinterpret_cast<const double2*>(T), reinterpret_cast<double2*>(V),
                   reinterpret_cast<const double2*>(VH), up_dst, reinterpret_cast<double2*>(lv_smem));
  } else {
    if (UP)
      k1_real_item(it, box, T_off, T, V, VH, up_dst, reinterpret_cast<double*>(lv_smem));
    else
      k3_real_item(it, box, T_off, T, V, VH, up_dst, reinterpret_cast<double*>(lv_smem));
  }
}

// ---- persistent tree passes (small, launch-bound plans) --------------------
// One launch runs the whole upward pass (K0, then every level deepest first)
// or the whole downward pass (every level coarsest first, then K4).  CTAs
// claim jobs in stage order from a counter; a job of stage s waits until the
// finished-job counter reaches the number of jobs in stages < s.  Jobs of
// stage >= s cannot start before that, so the count is reached exactly when
// every earlier stage is complete (empty stages included).  Deadlock-free:
// every job waited on was claimed earlier by a running CTA.  Same arithmetic
// as the per-level kernels (bit-identical).
struct TreePassArgs {
  const TreeJob* jobs;
  int64_t n_jobs;
  const int32_t* stage_first;  // jobs in the stages before stage s
  int* counter;
  int* done;                    // finished jobs
  const LevelItem* items;
  const int32_t* copy_boxes;
  const BoxRec* box;
  const int64_t* T_off;
  const double* T;
  const int32_t *slot, *orig, *hat, *up_dst;
  int64_t n_points;
  const double* q;  // up: charges in
  double* u;        // down: potentials out
  double *Q, *QH, *U, *UH;
};

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <class S, bool UP>
__global__ void __launch_bounds__(kUpThreads) k_tree_persist(TreePassArgs a) {
  static_assert(kUpThreads == kDownCols, "one block shape for K1 and K3 items");
  extern __shared__ __align__(16) unsigned char tp_smem[];
  S* sm = reinterpret_cast<S*>(tp_smem);
  __shared__ int s_job;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_job = atomicAdd(a.counter, 1);
    __syncthreads();
    const int64_t jn = s_job;
    if (jn >= a.n_jobs) return;
    const TreeJob job = a.jobs[jn];
    if (job.stage > 0 && threadIdx.x == 0)
      while (ld_acquire_i32(a.done) < a.stage_first[job.stage]) __nanosleep(32);
    __syncthreads();
    if (job.kind == kJobGather || job.kind == kJobScatter) {
      const int64_t t0 = (int64_t)job.a * kPointsPerJob;
      const int64_t t1 = t0 + kPointsPerJob < a.n_points ? t0 + kPointsPerJob : a.n_points;
      for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        if (UP)
          k0_point<S>(t, a.slot, a.orig, a.hat, a.up_dst, reinterpret_cast<const S*>(a.q),
                      reinterpret_cast<S*>(a.Q), reinterpret_cast<S*>(a.QH));
        else
          k4_point<S>(t, a.slot, a.orig, a.hat, a.up_dst, reinterpret_cast<const S*>(a.U),
                      reinterpret_cast<const S*>(a.UH), reinterpret_cast<S*>(a.u));
      }
    } else if (job.kind == kJobCopy) {
      if (warp < job.b) {
        const int32_t b = a.copy_boxes[job.a + warp];
        const S* Tb = reinterpret_cast<const S*>(a.T) + a.T_off[b];
        if (UP)
          k1_copy_box<S>(a.box[b], lane, Tb, reinterpret_cast<S*>(a.Q), reinterpret_cast<S*>(a.QH),
                         a.up_dst);
        else
          k3_copy_box<S>(a.box[b], lane, Tb, reinterpret_cast<S*>(a.U),
                         reinterpret_cast<const S*>(a.UH), a.up_dst);
      }
    } else {
      const LevelItem it = a.items[job.a];
      if constexpr (sizeof(S) == 16) {
        if (UP)
          k1_cplx_item(it, a.box, a.T_off, reinterpret_cast<const double2*>(a.T),
                       reinterpret_cast<double2*>(a.Q), reinterpret_cast<double2*>(a.QH), a.up_dst,
                       reinterpret_cast<double2*>(sm));
        else
          k3_cplx_item(it, a.box, a.T_off, reinterpret_cast<const double2*>(a.T),
                       reinterpret_cast<double2*>(a.U), reinterpret_cast<const double2*>(a.UH),
                       a.up_dst, reinterpret_cast<double2*>(sm));
      } else {
        if (UP)
          k1_real_item(it, a.box, a.T_off, a.T, a.Q, a.QH, a.up_dst, reinterpret_cast<double*>(sm));
        else
          k3_real_item(it, a.box, a.T_off, a.T, a.U, a.UH, a.up_dst, reinterpret_cast<double*>(sm));
      }
    }
    // publish this job's writes, then count it into its stage
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(a.done, 1);
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

}  // namespace

void launch_gather(const DevPlan& p, const double* q, DevState& s, cudaStream_t st) {
  const int g = grid_for(p.n_owned_points, 256);
  if (p.cplx)
    k0_gather<double2><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.leaf_hat, p.up_dst,
                                          p.n_owned_points, reinterpret_cast<const double2*>(q),
                                          reinterpret_cast<double2*>(s.Q),
                                          reinterpret_cast<double2*>(s.QH));
  else
    k0_gather<double><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.leaf_hat, p.up_dst,
                                         p.n_owned_points, q, s.Q, s.QH);
}

void launch_invert_orig(const DevPlan& p, int32_t* pos, cudaStream_t st) {
  k_invert_orig<<<grid_for(p.n_owned_points, 256), 256, 0, st>>>(p.leaf_orig, p.n_owned_points, pos);
}

void launch_scatter(const DevPlan& p, const DevState& s, double* u, cudaStream_t st) {
  const int g = grid_for(p.n_owned_points, 256);
  if (p.leaf_pos) {  // two passes, the fold staged in Q (free after the upward pass)
    if (p.cplx) {
      k4_fold<double2><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_hat, p.up_dst, p.n_owned_points,
                                          reinterpret_cast<const double2*>(s.U),
                                          reinterpret_cast<const double2*>(s.UH),
                                          reinterpret_cast<double2*>(s.Q));
      k4_gather<double2><<<g, 256, 0, st>>>(p.leaf_pos, p.n_owned_points,
                                            reinterpret_cast<const double2*>(s.Q),
                                            reinterpret_cast<double2*>(u));
    } else {
      k4_fold<double><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_hat, p.up_dst, p.n_owned_points, s.U,
                                         s.UH, s.Q);
      k4_gather<double><<<g, 256, 0, st>>>(p.leaf_pos, p.n_owned_points, s.Q, u);
    }
    return;
  }
  if (p.cplx)
    k4_scatter<double2><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.leaf_hat, p.up_dst,
                                           p.n_owned_points, reinterpret_cast<const double2*>(s.U),
                                           reinterpret_cast<const double2*>(s.UH),
                                           reinterpret_cast<double2*>(u));
  else
    k4_scatter<double><<<g, 256, 0, st>>>(p.leaf_slot, p.leaf_orig, p.leaf_hat, p.up_dst,
                                          p.n_owned_points, s.U, s.UH, u);
}

void launch_upward(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                   cudaStream_t st) {
  const int64_t c0 = hp.copy_lvl[level], c1 = hp.copy_lvl[level + 1];
  const int64_t j0 = hp.up1_lvl[level], j1 = hp.up1_lvl[level + 1];
  if (SFMM_K1_MERGE && c1 > c0 && j1 > j0 && !p.k1_bulk) {  // both kinds of work: one launch
    const int ncb = (int)((c1 - c0 + 7) / 8);
    const unsigned g = (unsigned)(ncb + (j1 - j0));
    if (p.cplx)
      k_level<double2, true><<<g, kUpThreads, p.up_smem, st>>>(
          p.copy_boxes + c0, c1 - c0, ncb, p.up1_items + j0, p.box, p.T_off, p.T, s.Q, s.QH, p.up_dst);
    else
      k_level<double, true><<<g, kUpThreads, p.up_smem, st>>>(
          p.copy_boxes + c0, c1 - c0, ncb, p.up1_items + j0, p.box, p.T_off, p.T, s.Q, s.QH, p.up_dst);
    return;
  }
  if (c1 > c0) {
    const unsigned g = (unsigned)((c1 - c0 + 7) / 8);
    if (p.cplx)
      k1_copy<double2><<<g, 256, 0, st>>>(p.copy_boxes + c0, c1 - c0, p.box, p.T_off,
                                          reinterpret_cast<const double2*>(p.T),
                                          reinterpret_cast<double2*>(s.Q),
                                          reinterpret_cast<double2*>(s.QH), p.up_dst);
    else
      k1_copy<double><<<g, 256, 0, st>>>(p.copy_boxes + c0, c1 - c0, p.box, p.T_off, p.T, s.Q, s.QH,
                                         p.up_dst);
  }
  const int64_t i0 = hp.up1_lvl[level], i1 = hp.up1_lvl[level + 1];
  if (i1 <= i0) return;
  if (p.cplx)
    k1_upward_cplx<<<(unsigned)(i1 - i0), kUpThreads, p.up_smem, st>>>(
        p.up1_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.Q), reinterpret_cast<double2*>(s.QH), p.up_dst);
  else if (p.k1_bulk)
    k1_upward_real_bulk<<<(unsigned)std::min<int64_t>(i1 - i0, p.k1_bulk_grid), kK1BulkThreads,
                          p.up_bulk_smem, st>>>(p.up1_items + i0, i1 - i0, p.box, p.T_off, p.T,
                                                s.Q, s.QH, p.up_dst, p.up_bulk_qr);
  else
    k1_upward_real<<<(unsigned)(i1 - i0), kUpThreads, p.up_smem, st>>>(
        p.up1_items + i0, p.box, p.T_off, p.T, s.Q, s.QH, p.up_dst);
}

void launch_downward(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                     cudaStream_t st) {
  const int64_t c0 = hp.copy_dn_lvl[level], c1 = hp.copy_dn_lvl[level + 1];
  const int64_t j0 = hp.down_lvl[level], j1 = hp.down_lvl[level + 1];
  // (SFMM_K3_MERGE, plan_build.h: off -- the merged downward launch measured
  // slower on adaptive trees, config 3a 1.42 vs 1.36 ms, 3b 2.47 vs 2.35 ms)
  if (SFMM_K3_MERGE && c1 > c0 && j1 > j0) {  // both kinds of work: one launch
    const int ncb = (int)((c1 - c0 + 7) / 8);
    const unsigned g = (unsigned)(ncb + (j1 - j0));
    if (p.cplx)
      k_level<double2, false><<<g, kDownCols, p.down_smem, st>>>(
          p.copy_boxes_dn + c0, c1 - c0, ncb, p.down_items + j0, p.box, p.T_off, p.T, s.U, s.UH, p.up_dst);
    else
      k_level<double, false><<<g, kDownCols, p.down_smem, st>>>(
          p.copy_boxes_dn + c0, c1 - c0, ncb, p.down_items + j0, p.box, p.T_off, p.T, s.U, s.UH, p.up_dst);
    return;
  }
  if (c1 > c0) {
    const unsigned g = (unsigned)((c1 - c0 + 7) / 8);
    if (p.cplx)
      k3_copy<double2><<<g, 256, 0, st>>>(p.copy_boxes_dn + c0, c1 - c0, p.box, p.T_off,
                                          reinterpret_cast<const double2*>(p.T),
                                          reinterpret_cast<double2*>(s.U),
                                          reinterpret_cast<const double2*>(s.UH), p.up_dst);
    else
      k3_copy<double><<<g, 256, 0, st>>>(p.copy_boxes_dn + c0, c1 - c0, p.box, p.T_off, p.T, s.U, s.UH,
                                         p.up_dst);
  }
  const int64_t i0 = hp.down_lvl[level], i1 = hp.down_lvl[level + 1];
  if (i1 <= i0) return;
  if (p.cplx)
    k3_downward_cplx<<<(unsigned)(i1 - i0), kDownCols, p.down_smem, st>>>(
        p.down_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.U), reinterpret_cast<const double2*>(s.UH), p.up_dst);
  else
    k3_downward_real<<<(unsigned)(i1 - i0), kDownCols, p.down_smem, st>>>(
        p.down_items + i0, p.box, p.T_off, p.T, s.U, s.UH, p.up_dst);
}

namespace {

TreePassArgs tree_args(const DevPlan& p, bool up, const DevState& s) {
  TreePassArgs a;
  a.jobs = up ? p.up_jobs : p.down_jobs;
  a.n_jobs = up ? p.n_up_jobs : p.n_down_jobs;
  a.stage_first = up ? p.up_stage_first : p.down_stage_first;
  a.counter = p.tree_sync + (up ? 0 : 1);
  a.done = p.tree_sync + (up ? 2 : 3);
  a.items = up ? p.up1_items : p.down_items;
  a.copy_boxes = up ? p.copy_boxes : p.copy_boxes_dn;
  a.box = p.box;
  a.T_off = p.T_off;
  a.T = p.T;
  a.slot = p.leaf_slot;
  a.orig = p.leaf_orig;
  a.hat = p.leaf_hat;
  a.up_dst = p.up_dst;
  a.n_points = p.n_owned_points;
  a.q = nullptr;
  a.u = nullptr;
  a.Q = s.Q;
  a.QH = s.QH;
  a.U = s.U;
  a.UH = s.UH;
  return a;
}

}  // namespace

void launch_upward_all(const DevPlan& p, const HostPlan& hp, const double* q, DevState& s,
                       cudaStream_t st) {
  if (!p.tree_persist) {
    launch_gather(p, q, s, st);
    for (int l = hp.depth; l >= 2; --l) launch_upward(p, hp, l, s, st);
    return;
  }
  // counters and done flags of both passes (the downward launch follows K2)
  cudaMemsetAsync(p.tree_sync, 0, sizeof(int) * 4, st);
  TreePassArgs a = tree_args(p, true, s);
  a.q = q;
  const unsigned g = (unsigned)std::min<int64_t>(p.persist_grid, std::max<int64_t>(p.n_up_jobs, 1));
  if (p.cplx)
    k_tree_persist<double2, true><<<g, kUpThreads, p.persist_smem, st>>>(a);
  else
    k_tree_persist<double, true><<<g, kUpThreads, p.persist_smem, st>>>(a);
}

void launch_downward_all(const DevPlan& p, const HostPlan& hp, DevState& s, double* u,
                         cudaStream_t st) {
  if (!p.tree_persist) {
    for (int l = 2; l <= hp.depth; ++l) launch_downward(p, hp, l, s, st);
    launch_scatter(p, s, u, st);
    return;
  }
  TreePassArgs a = tree_args(p, false, s);
  a.u = u;
  const unsigned g = (unsigned)std::min<int64_t>(p.persist_grid, std::max<int64_t>(p.n_down_jobs, 1));
  if (p.cplx)
    k_tree_persist<double2, false><<<g, kUpThreads, p.persist_smem, st>>>(a);
  else
    k_tree_persist<double, false><<<g, kUpThreads, p.persist_smem, st>>>(a);
}

void launch_direct_fallback(const DevPlan& p, const double* q, double* u, cudaStream_t st) {
  const int threads = 128;
  const unsigned g = (unsigned)((p.n_points + threads - 1) / threads);
  k5_direct<<<g, threads, 0, st>>>(p.kernel, p.kappa, p.dim, p.cplx, p.n_points, p.orig_pts, q,
                                   u, p.err_flag);
}

void launch_direct_subset(int kernel, double kappa, int dim, int64_t n, const double* pts,
                          const double* q, int64_t nt, const int32_t* targets, double* u,
                          int* err_flag, cudaStream_t st) {
  if (nt <= 0) return;
  k5_direct_subset<<<(unsigned)nt, 256, 0, st>>>(kernel, kappa, dim,
                                                 kernel == SFMM_HELMHOLTZ3D ? 1 : 0, n, pts, q,
                                                 targets, u, err_flag);
}

namespace {

// Ghost exchange: element i of the buffer <-> [Q | QH][idx[i]] (QH addressed
// from n_slots on).  One thread per element, coalesced on the buffer side.
template <class S, bool kPack>
__global__ void k_exchange(const int64_t* __restrict__ idx, int64_t n, int64_t n_slots,
                           S* __restrict__ Q, S* __restrict__ QH, S* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx[i];
    S* p = k < n_slots ? Q + k : QH + (k - n_slots);
    if (kPack)
      buf[i] = *p;
    else
      *p = buf[i];
  }
}

__device__ __forceinline__ double xadd(double a, double b) { return a + b; }
__device__ __forceinline__ double2 xadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}

// Second exchange: one CTA per (peer, receiving box) group sums the group's
// staged column sums over its row tiles (fixed tile order) into the send
// buffer.  The tile offsets are staged in shared memory first so the value
// loads of several tiles are in flight at once (the adds stay in order).
template <class S>
__global__ void __launch_bounds__(256) k_xpack(const int64_t* __restrict__ tile_off,
                                               const int64_t* __restrict__ tile_u,
                                               const int64_t* __restrict__ tile_h,
                                               const int64_t* __restrict__ dst,
                                               const int32_t* __restrict__ nu,
                                               const int32_t* __restrict__ nh,
                                               const S* __restrict__ St, S* __restrict__ buf) {
  constexpr int kT = 128;  // tiles staged per round
  __shared__ int64_t su[kT], sh[kT];
  const int64_t i = blockIdx.x, t0 = tile_off[i], t1 = tile_off[i + 1];
  const int n_u = nu[i], n = n_u + nh[i];
  S* out = buf + dst[i];
  for (int j0 = 0; j0 < n; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    S s = S{};
    for (int64_t c0 = t0; c0 < t1; c0 += kT) {
      const int cnt = (int)(t1 - c0 < kT ? t1 - c0 : kT);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        su[t] = tile_u[c0 + t];
        sh[t] = tile_h[c0 + t];
      }
      __syncthreads();
      if (j < n) {
        if (j < n_u) {
#pragma unroll 4
          for (int t = 0; t < cnt; ++t) s = xadd(s, St[su[t] + j]);
        } else {
#pragma unroll 4
          for (int t = 0; t < cnt; ++t)
            if (sh[t] >= 0) s = xadd(s, St[sh[t] + (j - n_u)]);
        }
      }
    }
    if (j < n) out[j] = s;
  }
}

}  // namespace

void launch_xpack(const DevPlan& p, double* buf, cudaStream_t st) {
  if (p.n_xpairs == 0) return;
  if (p.cplx)
    k_xpack<double2><<<(unsigned)p.n_xpairs, 256, 0, st>>>(
        p.xpair_tile_off, p.xtile_u, p.xtile_h, p.xpair_dst, p.xpair_nu, p.xpair_nh,
        reinterpret_cast<const double2*>(p.stage), reinterpret_cast<double2*>(buf));
  else
    k_xpack<double><<<(unsigned)p.n_xpairs, 256, 0, st>>>(p.xpair_tile_off, p.xtile_u, p.xtile_h,
                                                           p.xpair_dst, p.xpair_nu, p.xpair_nh,
                                                           p.stage, buf);
}

void launch_pack(const DevPlan& p, const DevState& s, double* buf, cudaStream_t st) {
  if (p.n_pack == 0) return;
  const int g = grid_for(p.n_pack, 256);
  if (p.cplx)
    k_exchange<double2, true><<<g, 256, 0, st>>>(p.pack_idx, p.n_pack, p.n_slots,
                                                  reinterpret_cast<double2*>(s.Q),
                                                  reinterpret_cast<double2*>(s.QH),
                                                  reinterpret_cast<double2*>(buf));
  else
    k_exchange<double, true><<<g, 256, 0, st>>>(p.pack_idx, p.n_pack, p.n_slots, s.Q, s.QH, buf);
}

void launch_unpack(const DevPlan& p, DevState& s, const double* buf, cudaStream_t st) {
  if (p.n_unpack == 0) return;
  const int g = grid_for(p.n_unpack, 256);
  double* b = const_cast<double*>(buf);
  if (p.cplx)
    k_exchange<double2, false><<<g, 256, 0, st>>>(p.unpack_idx, p.n_unpack, p.n_slots,
                                                   reinterpret_cast<double2*>(s.Q),
                                                   reinterpret_cast<double2*>(s.QH),
                                                   reinterpret_cast<double2*>(b));
  else
    k_exchange<double, false><<<g, 256, 0, st>>>(p.unpack_idx, p.n_unpack, p.n_slots, s.Q, s.QH, b);
}

int configure_tree_kernels(DevPlan& p, size_t max_r, size_t max_k) {
  const size_t sw = p.cplx ? 16 : 8;
  p.up_smem = std::max<size_t>(max_r * sw, 16);
  if (p.up_smem > 48 * 1024 &&
      cudaFuncSetAttribute(p.cplx ? (const void*)k1_upward_cplx : (const void*)k1_upward_real,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.up_smem) != cudaSuccess)
    return -1;
  // real K1 through the bulk-copy ring (opt-in A/B: SFMM_K1_BULK=1; measured
  // slower than the register stream) when every T row fits a stage
  p.k1_bulk = 0;
  if (!p.cplx && max_r <= (size_t)kK1MaxR && std::getenv("SFMM_K1_BULK")) {
    p.up_bulk_qr = (int)(((max_r + 2) + 1) & ~(size_t)1);  // q_R doubles per stage (16-byte multiple)
    p.up_bulk_smem = 128 + 64 * kK1Stages +
                     (size_t)kK1Stages * ((size_t)kK1StageBytes + 8 * (size_t)p.up_bulk_qr);
    if (cudaFuncSetAttribute((const void*)k1_upward_real_bulk,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p.up_bulk_smem) != cudaSuccess)
      return -1;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p.k1_bulk_grid = sms;  // one persistent CTA per SM (the ring takes ~160 KB)
    p.k1_bulk = 1;
  }
  if (p.tree_persist) {
    p.persist_smem = std::max(p.up_smem, std::max<size_t>(max_k * sw, 16));
    const void* f[4] = {(const void*)k_tree_persist<double, true>,
                        (const void*)k_tree_persist<double, false>,
                        (const void*)k_tree_persist<double2, true>,
                        (const void*)k_tree_persist<double2, false>};
    int per_sm = 0, dev = 0, sms = 148;
    for (const void* fn : f)
      if (p.persist_smem > 48 * 1024 &&
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)p.persist_smem) != cudaSuccess)
        return -1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, p.cplx ? (const void*)k_tree_persist<double2, true>
                            : (const void*)k_tree_persist<double, true>,
            kUpThreads, p.persist_smem) != cudaSuccess)
      return -1;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p.persist_grid = sms * std::max(1, per_sm);
  }
  if (p.up_smem > 48 * 1024 &&
      cudaFuncSetAttribute(p.cplx ? (const void*)k_level<double2, true> : (const void*)k_level<double, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.up_smem) != cudaSuccess)
    return -1;
  p.down_smem = std::max<size_t>(max_k * sw, 16);
  if (p.down_smem > 48 * 1024 &&
      cudaFuncSetAttribute(p.cplx ? (const void*)k_level<double2, false> : (const void*)k_level<double, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.down_smem) != cudaSuccess)
    return -1;
  if (p.down_smem > 48 * 1024) {
    if (cudaFuncSetAttribute(
            p.cplx ? (const void*)k3_downward_cplx : (const void*)k3_downward_real,
            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.down_smem) != cudaSuccess)
      return -1;
  }
  return 0;
}

void launch_build_slots(const SlotBuildArgs& a, cudaStream_t st) {
  constexpr int kThreads = 256, kWarps = kThreads / 32;
  if (a.n_boxes > 0)
    k_build_slots<<<(int)((a.n_boxes + kWarps - 1) / kWarps), kThreads, 0, st>>>(a);
  if (a.n_leaves > 0)
    k_build_leaf_maps<<<(int)((a.n_leaves + kWarps - 1) / kWarps), kThreads, 0, st>>>(a);
}

}  // namespace sfmm_gpu
