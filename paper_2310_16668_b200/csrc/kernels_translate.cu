// K2: the fused translation kernel (ifo + ifs + tfo + level-1 in one launch).
//
// Replaces translate_ifo / translate_ifs / translate_tfo / level1_dense and
// their microkernel add_block (/root/reference/proj/src/apply.cpp:16-42,
// :148-266).  The reference generates every kernel entry G(x_i, x_j) on the
// fly for each (target box, source box) pair and runs a second, skeleton-only
// add_block for the subtract term.  Here every subtract term is folded into
// the dense pass: S_b is a subset of B_b with the same ids, so G is generated
// once per (row i, source j) and accumulated into
//     acc_u += G * a_j        (a_j = q_j, or q_j - qhat_j for tfo)
//     acc_h += G * h_j        (h_j = qhat_j on skeleton slots for ifo, q_j for
//                              ifs; only for tasks that own skeleton rows)
// and the results are stored once per row: U = acc_u * c, UH = -acc_h * c.
//
// Scheduling: persistent warps pull cost-sorted tasks (box, 128-row tile)
// from an atomic counter.  Each row is owned by exactly one warp, so outputs
// are plain stores: no result atomics, deterministic, thread-count
// independent (apply.hpp:88-90).  Sources are staged per warp through shared
// memory in chunks of 32 and broadcast to every lane; each lane holds up to
// four target rows in registers.
//
// The zero diagonal (apply.cpp:31-34) is applied by index in self blocks.  A
// coincident pair with distinct ids makes the generated entry non-finite; a
// non-finite row result triggers an exact re-scan of that row, which raises
// the duplicate flag only if such a pair exists (NaN charges stay NaN, as in
// the reference).
#include <math.h>

#include <algorithm>

#include "fastmath.cuh"
#include "launch.h"

namespace sfmm_gpu {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr unsigned kFull = 0xffffffffu;
constexpr double kInv4Pi = 0.0795774715459476678844418816862571810;  // 1/(4 pi)

struct K2Args {
  const BoxRec* box;
  const EntryRange* er;
  const int32_t* ent;
  const Task* tasks;
  int64_t n_tasks;
  const double *X, *Y, *Z;
  const int32_t* sid;
  const double* Q;
  const double* QH;
  double* U;
  double* UH;
  int* counter;
  int* err;
  double kappa;
  double* St;  // staging for kSYM column sums (unscaled)
  unsigned* sflag;  // per 32 staged scalars: row tiles of the box that have added (chaining)
  const double2* tab;  // (cos, sin)(k pi/128), Helmholtz only
  const double* ltab;  // log table (fastmath.cuh), Laplace 2D only
};

// Far-away padding for partial source chunks of kSYM blocks: finite r^2,
// negligible G, zero weights.
constexpr double kFar = 1e100;

// rsqrt to full double precision: MUFU.RSQ64H seed + one cubic correction
// (5 FP64 ops).  r2 == 0 yields NaN, which the diagonal select / duplicate
// check handle.
__device__ __forceinline__ double rsqrt_fp64(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double h = y * y;
  const double e = fma(-r2, h, 1.0);
  const double p = fma(0.375, e, 0.5);
  const double ye = y * e;
  return fma(p, ye, y);
}

// Real kernels: g(r2) is proportional to G; the constant goes into `scale`.
struct GenLaplace3d {  // kernel.hpp:46-50  1/(4 pi r)
  static constexpr int kDim = 3;
  static constexpr double kScale = kInv4Pi;
  static constexpr bool kLogTable = false;
  __device__ static __forceinline__ double g(double r2, uint32_t) { return rsqrt_fp64(r2); }
  // M independent evaluations, stage by stage, so their dependent chains
  // interleave in the issue stream.
  template <int M>
  __device__ static __forceinline__ void batch(const double* r2, double* g, uint32_t) {
    double y[M], e[M];
#pragma unroll
    for (int m = 0; m < M; ++m) asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[m]) : "d"(r2[m]));
#pragma unroll
    for (int m = 0; m < M; ++m) e[m] = fma(-r2[m], y[m] * y[m], 1.0);
#pragma unroll
    for (int m = 0; m < M; ++m) g[m] = fma(fma(0.375, e[m], 0.5), y[m] * e[m], y[m]);
  }
};
struct GenLaplace2d {  // kernel.hpp:40-44  -log(r^2)/(4 pi)
  static constexpr int kDim = 2;
  static constexpr double kScale = -kInv4Pi;
  static constexpr bool kLogTable = true;  // log_tab with the table in shared memory
  __device__ static __forceinline__ double g(double r2, uint32_t lt) { return log_tab(lt, r2); }
  template <int M>
  __device__ static __forceinline__ void batch(const double* r2, double* g, uint32_t lt) {
#pragma unroll
    for (int m = 0; m < M; ++m) g[m] = log_tab(lt, r2[m]);
  }
};

struct WarpSmemReal {
  double2 xy[32];
  double2 za[32];  // z, a-weight
  double h[32];
  // per-tile layout: the rotation's starting column sums (a merged task's
  // later tiles: the earlier tiles' sums of the pair's staged vector, else 0)
  double pu[32], ph[32];
  unsigned* fbase;  // chain flags of the current kSYM entry (kept out of registers)
  int tile;
  // the current tile of the task (merged tasks: one of the box's tiles) and
  // the merged task's next tile, kept out of registers
  int row0, nrows, pend_t, pend_r0;
};

struct WarpSmemCplx {
  double2 xy[32];
  double z[32];
  double2 a[32];
  double2 h[32];
  unsigned* fbase;
  int tile;
  int row0, nrows, pend_t, pend_r0;
};

// Chained kSYM column sums: the row tiles of a box add their column sums of a
// pair (b, c) into ONE staged vector, in tile order.  Tile t waits until the
// chunk's flag says t tiles have added, adds its partial sums to the staged
// ones (read through L2), stores, and publishes t + 1.  Tiles of one box are
// claimed from the task counter in tile order (plan_build.cpp keeps them in
// that order), so tile t - 1 is always running or done: no circular wait.
// The order of the additions is fixed, so results stay deterministic.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double add_s(double a, double b) { return a + b; }

__device__ __forceinline__ double2 add_s(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
template <class S, bool H, bool CHAIN>
__device__ __forceinline__ void chain_store(S* st_u, S* st_h, S cp, S ch, int col, int n_c,
                                            int k_c, const unsigned* const* fbase, const int* tilep,
                                            int j0, int lane) {
  if constexpr (!CHAIN) {  // this tile's own staged vector (merged tasks: see sym_chunk)
    if (col < n_c) st_u[col] = cp;
    if (H && col < k_c) st_h[col] = ch;
    return;
  }
  unsigned* flag = const_cast<unsigned*>(*fbase) + (j0 >> 5);
  const int tile = *tilep;
  if (tile > 0) {
    while (ld_acquire_u32(flag) < (unsigned)tile) __nanosleep(32);
    if (col < n_c) cp = add_s(__ldcg(st_u + col), cp);
    if (H && col < k_c) ch = add_s(__ldcg(st_h + col), ch);
  }
  if (col < n_c) __stcg(st_u + col, cp);
  if (H && col < k_c) __stcg(st_h + col, ch);
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release_u32(flag, (unsigned)tile + 1);
}

// Exact re-scan of one row for coincident points with distinct ids.
__device__ __noinline__ void verify_row(const K2Args& a, int32_t b, int32_t row, int dim) {
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
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (r2 == 0.0 && a.sid[t] != id) atomicOr(a.err, 1);
    }
  }
}

template <class G, int R, bool H, bool SELF>
__device__ __forceinline__ void inner_real(const WarpSmemReal& sm, uint32_t lt, int cnt, int j0,
                                           const double (&xi)[R], const double (&yi)[R],
                                           const double (&zi)[R], const int (&rowi)[R],
                                           double (&au)[R], double (&ah)[R]) {
#pragma unroll 2
  for (int jj = 0; jj < cnt; ++jj) {
    const double2 xy = sm.xy[jj];
    const double2 za = sm.za[jj];
    const double wh = H ? sm.h[jj] : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = xi[r] - xy.x;
      const double dy = yi[r] - xy.y;
      double r2 = fma(dy, dy, dx * dx);
      if (G::kDim == 3) {
        const double dz = zi[r] - za.x;
        r2 = fma(dz, dz, r2);
      }
      double g = G::g(r2, lt);
      if (SELF) g = (rowi[r] == j0 + jj) ? 0.0 : g;
      au[r] = fma(g, za.y, au[r]);
      if (H) ah[r] = fma(g, wh, ah[r]);
    }
  }
}

// One staged source chunk of a kSYM block: b's rows (registers) against 32 of
// c's columns.  Row sums as for kIFO.  Column sums sum_i G(i,j) q_b[i] (and,
// with H, sum_{i<k_b} G(i,j) qhat_b[i] for j < k_c) use a rotation instead of a
// reduction: at step s lane l evaluates column (l+s) mod 32 for its R rows and
// the running column sum moves one lane down, so after 32 steps lane l holds
// the complete sum of column l over the warp's 32R rows.  Fixed order, no
// butterfly, two column accumulators per lane.
template <class G, int R, bool H, bool CHAIN, bool MERGE>
__device__ __forceinline__ void sym_chunk(const WarpSmemReal& sm, uint32_t lt, int j0, int n_c,
                                          int k_c,
                                          const double (&xi)[R], const double (&yi)[R],
                                          const double (&zi)[R], const double (&qr)[R],
                                          const double (&qhr)[R], double (&au)[R],
                                          double (&ah)[R], double* __restrict__ st_u,
                                          double* __restrict__ st_h, int lane) {
  double cp = 0.0, ch = 0.0;
  // a merged task's later tiles start the rotation from the earlier tiles'
  // sums of their column (stored by this same thread: the running sum ends
  // in the lane it started in), so the pair keeps one staged vector
  if (MERGE) {
    cp = sm.pu[lane];
    if (H) ch = sm.ph[lane];
  }
  const int from = (lane + 1) & 31;
#pragma unroll 4
  for (int s = 0; s < 32; ++s) {
    const int jc = (lane + s) & 31;
    const double2 xy = sm.xy[jc];
    const double2 za = sm.za[jc];
    const double wh = H ? sm.h[jc] : 0.0;
    double r2[R], g[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = xi[r] - xy.x;
      const double dy = yi[r] - xy.y;
      r2[r] = fma(dy, dy, dx * dx);
      if (G::kDim == 3) {
        const double dz = zi[r] - za.x;
        r2[r] = fma(dz, dz, r2[r]);
      }
    }
    G::template batch<R>(r2, g, lt);
    double cs = 0.0, hs = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      au[r] = fma(g[r], za.y, au[r]);
      cs = fma(g[r], qr[r], cs);
      if (H) {
        ah[r] = fma(g[r], wh, ah[r]);
        hs = fma(g[r], qhr[r], hs);
      }
    }
    cp = __shfl_sync(kFull, cp + cs, from);
    if (H) ch = __shfl_sync(kFull, ch + hs, from);
  }
  chain_store<double, H, CHAIN>(st_u, st_h, cp, ch, j0 + lane, n_c, k_c, &sm.fbase, &sm.tile, j0,
                                lane);
}

// Rows [row0, row0 + nrows) of task t: the task's tile, or one tile of a
// merged task (all row tiles of a box in one task, plan_build.cpp), whose
// kSYM column sums share one staged vector per pair (as the chained layout).
template <class G, int R, bool CHAIN, bool MERGE>
__device__ __forceinline__ void task_real(const K2Args& a, const Task& t, WarpSmemReal& sm,
                                          uint32_t lt, int lane) {
  const int row0 = MERGE ? sm.row0 : t.row0;
  const BoxRec tb = a.box[t.box];
  double xi[R], yi[R], zi[R], au[R], ah[R], qr[R], qhr[R];
  int rowi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = row0 + r * 32 + lane;
    rowi[r] = row;
    const bool valid = row < row0 + (MERGE ? sm.nrows : t.nrows);
    const int64_t s = tb.slot + (valid ? row : row0);
    xi[r] = a.X[s];
    yi[r] = a.Y[s];
    zi[r] = G::kDim == 3 ? a.Z[s] : 0.0;
    qr[r] = valid ? a.Q[s] : 0.0;  // row charges feed kSYM column sums
    qhr[r] = (valid && row < tb.k) ? a.QH[tb.skel + row] : 0.0;
    au[r] = 0.0;
    ah[r] = 0.0;
  }
  const EntryRange er = a.er[t.box];
  const bool skel_rows = row0 < tb.k;
  // one staged vector per pair for every row tile: chained or merged layout
  const bool pair_stage = CHAIN || (MERGE && t.nrows > sm.nrows);
  int64_t stage = t.stage;
  const int e_end = t.e1 < 0 ? er.count : t.e1;
  for (int e = t.e0; e < e_end; ++e) {
    const int32_t code = a.ent[er.begin + e];
    const int32_t c = code >> kModeBits;
    const int mode = code & kModeMask;
    const BoxRec sb = a.box[c];
    if (mode == kSYM) {
      double* st_u = a.St + stage;
      double* st_h = st_u + sb.n;
      if (CHAIN && lane == 0) {
        sm.fbase = a.sflag + (stage >> 5);
        sm.tile = t.tile;
      }
      for (int j0 = 0; j0 < sb.n; j0 += 32) {
        const int j = j0 + lane;
        if (j < sb.n) {
          const int64_t s = sb.slot + j;
          sm.xy[lane] = make_double2(a.X[s], a.Y[s]);
          sm.za[lane] = make_double2(G::kDim == 3 ? a.Z[s] : 0.0, a.Q[s]);
          sm.h[lane] = j < sb.k ? a.QH[sb.skel + j] : 0.0;
        } else {
          sm.xy[lane] = make_double2(kFar, kFar);
          sm.za[lane] = make_double2(kFar, 0.0);
          sm.h[lane] = 0.0;
        }
        if (MERGE) {  // a merged task's later tiles continue the pair's sums
          const bool acc = sm.tile > 0;
          sm.pu[lane] = acc && j < sb.n ? st_u[j] : 0.0;
          sm.ph[lane] = acc && j < sb.k ? st_h[j] : 0.0;
        }
        __syncwarp();
        if (skel_rows && j0 < sb.k)
          sym_chunk<G, R, true, CHAIN, MERGE>(sm, lt, j0, sb.n, sb.k, xi, yi, zi, qr, qhr, au, ah, st_u, st_h,
                                lane);
        else
          sym_chunk<G, R, false, CHAIN, MERGE>(sm, lt, j0, sb.n, sb.k, xi, yi, zi, qr, qhr, au, ah, st_u, st_h,
                                 lane);
        __syncwarp();
      }
      stage += (sb.n + (((pair_stage ? tb.k > 0 : skel_rows) && sb.k > 0) ? sb.k : 0) + 31) &
               ~(int64_t)31;
      continue;
    }
    const bool self = c == t.box;
    for (int j0 = 0; j0 < sb.n; j0 += 32) {
      const int j = j0 + lane;
      if (j < sb.n) {
        const int64_t s = sb.slot + j;
        const double q = a.Q[s];
        const double qh = j < sb.k ? a.QH[sb.skel + j] : 0.0;
        double wa = q, wh = 0.0;
        if (mode == kIFO) wh = qh;
        else if (mode == kIFS) wh = q;
        else if (mode == kTFO) wa = q - qh;
        sm.xy[lane] = make_double2(a.X[s], a.Y[s]);
        sm.za[lane] = make_double2(G::kDim == 3 ? a.Z[s] : 0.0, wa);
        sm.h[lane] = wh;
      }
      __syncwarp();
      const int cnt = min(32, sb.n - j0);
      const bool need_h = skel_rows && (mode == kIFS || (mode == kIFO && j0 < sb.k));
      if (self) {
        if (need_h) inner_real<G, R, true, true>(sm, lt, cnt, j0, xi, yi, zi, rowi, au, ah);
        else inner_real<G, R, false, true>(sm, lt, cnt, j0, xi, yi, zi, rowi, au, ah);
      } else {
        if (need_h) inner_real<G, R, true, false>(sm, lt, cnt, j0, xi, yi, zi, rowi, au, ah);
        else inner_real<G, R, false, false>(sm, lt, cnt, j0, xi, yi, zi, rowi, au, ah);
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = rowi[r];
    if (row >= (MERGE ? sm.row0 + sm.nrows : t.row0 + t.nrows)) continue;
    const bool skel_row = row < tb.k;
    if (!isfinite(au[r]) || (skel_row && !isfinite(ah[r]))) verify_row(a, t.box, row, G::kDim);
    if constexpr (R == 1) {  // (only 32-row tiles are ever split, plan_build.cpp)
      if (t.rstage >= 0) {  // a later part of a split task: raw row partials, added by K2b
        a.St[t.rstage + row] = au[r];
        if (skel_row) a.St[t.rstage + tb.n + row] = ah[r];
        continue;
      }
    }
    a.U[tb.slot + row] = au[r] * G::kScale;
    if (skel_row) a.UH[tb.skel + row] = -ah[r] * G::kScale;
  }
}

#ifndef SFMM_K2_MIN_BLOCKS
#define SFMM_K2_MIN_BLOCKS 4
#endif
// Plans whose every task has <= 32 rows (small trees, config-1 sized) run a
// 1-row-per-lane instantiation capped at 64 registers: twice the resident
// warps to hide the dependent generation chains (the 128-register kernel
// carries the R = 4 variant's register budget).
#ifndef SFMM_K2_R1_MIN_BLOCKS
#define SFMM_K2_R1_MIN_BLOCKS 8
#endif
template <class G, int MAXR, int MINB, bool CHAIN, bool MERGE>
__global__ void __launch_bounds__(kThreads, MINB) k2_translate_real_t(K2Args a) {
  __shared__ WarpSmemReal smem[kWarps];
  __shared__ __align__(16) double ltab[G::kLogTable ? kLogTabLen : 1];
  if (G::kLogTable) {
    for (int i = threadIdx.x; i < kLogTabLen; i += blockDim.x) ltab[i] = a.ltab[i];
    __syncthreads();
  }
  const uint32_t lts = log_tab_addr(ltab);
  const int lane = threadIdx.x & 31;
  WarpSmemReal& sm = smem[threadIdx.x >> 5];
  if constexpr (MERGE) {
    if (lane == 0) sm.pend_t = -1;
    for (;;) {
      // the next tile: a merged task's next one (its box's row tiles in order,
      // plan_build.cpp), else a new task from the counter; the tile's rows
      // are handed over in shared memory (kept out of registers)
      int t = 0;
      if (lane == 0) {
        int r0 = 0;
        if (sm.pend_t >= 0) {
          t = sm.pend_t;
          r0 = sm.pend_r0;
        } else {
          t = atomicAdd(a.counter, 1);
        }
        sm.pend_t = -1;
        if (t < a.n_tasks) {
          constexpr int kTile = 32 * MAXR;
          const int nr = a.tasks[t].nrows;
          sm.row0 = a.tasks[t].row0 + r0;
          sm.nrows = min(kTile, nr - r0);
          sm.tile = r0 / kTile;
          if (r0 + kTile < nr) {
            sm.pend_t = t;
            sm.pend_r0 = r0 + kTile;
          }
        }
      }
      t = __shfl_sync(kFull, t, 0);  // (also orders lane 0's tile fields for the warp)
      if (t >= a.n_tasks) return;
      const Task& task = a.tasks[t];
      switch ((sm.nrows + 31) >> 5) {
        case 1: task_real<G, 1, false, true>(a, task, sm, lts, lane); break;
#if SFMM_K2_MAX_R >= 2
        case 2: task_real<G, 2, false, true>(a, task, sm, lts, lane); break;
#endif
#if SFMM_K2_MAX_R >= 3
        case 3: task_real<G, 3, false, true>(a, task, sm, lts, lane); break;
#endif
        default: task_real<G, MAXR, false, true>(a, task, sm, lts, lane); break;
      }
      __syncwarp();
    }
  } else {
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(a.counter, 1);
      t = __shfl_sync(kFull, t, 0);
      if (t >= a.n_tasks) return;
      // by reference: the task's fields are read where they are used instead of
      // being held in registers through the whole task (entry range, row-partial
      // slot of split tasks)
      const Task& task = a.tasks[t];
      if constexpr (MAXR == 1) {
        task_real<G, 1, CHAIN, false>(a, task, sm, lts, lane);
      } else {
        switch ((task.nrows + 31) >> 5) {
          case 1: task_real<G, 1, CHAIN, false>(a, task, sm, lts, lane); break;
#if SFMM_K2_MAX_R >= 2
          case 2: task_real<G, 2, CHAIN, false>(a, task, sm, lts, lane); break;
#endif
#if SFMM_K2_MAX_R >= 3
          case 3: task_real<G, 3, CHAIN, false>(a, task, sm, lts, lane); break;
#endif
          default: task_real<G, SFMM_K2_MAX_R, CHAIN, false>(a, task, sm, lts, lane); break;
        }
      }
    }
  }
}
template <class G>
constexpr auto k2_real_kernel(bool r1, bool chain, bool merged) {
  // merged plans (plan_build.cpp) have tasks of more than one tile: never r1 or chained
  if (merged) return k2_translate_real_t<G, SFMM_K2_MAX_R, SFMM_K2_MIN_BLOCKS, false, true>;
  return chain ? (r1 ? k2_translate_real_t<G, 1, SFMM_K2_R1_MIN_BLOCKS, true, false>
                     : k2_translate_real_t<G, SFMM_K2_MAX_R, SFMM_K2_MIN_BLOCKS, true, false>)
               : (r1 ? k2_translate_real_t<G, 1, SFMM_K2_R1_MIN_BLOCKS, false, false>
                     : k2_translate_real_t<G, SFMM_K2_MAX_R, SFMM_K2_MIN_BLOCKS, false, false>);
}

// ---------------------------------------------------------------------------
// Helmholtz 3D, complex FP64: G = exp(i kappa r)/(4 r) (kernel.hpp:62-71).
// ---------------------------------------------------------------------------
// Complex K2 shape (A/B at N=2e6, kappa=10, K2 ms): rows per lane <= 2 at
// 4 CTAs/SM 68.5; <= 3 at 3 CTAs/SM 66.1, plus two sources per loop trip 65.6
// (adopted); <= 4 at 3 CTAs/SM 69.1; <= 3 at 4 CTAs/SM (spills) 68.1.
#ifndef SFMM_K2C_UNROLL
#define SFMM_K2C_UNROLL 2
#endif
constexpr int kK2cUnroll = SFMM_K2C_UNROLL;
// rotation steps per loop trip in sym_chunk_cplx (A/B at 2e6, K2 ms: 2 63.2,
// 1 61.6, 4 65.5)
#ifndef SFMM_K2C_SYM_UNROLL
#define SFMM_K2C_SYM_UNROLL 1
#endif
constexpr int kSymCplxUnroll = SFMM_K2C_SYM_UNROLL;
template <int R, bool H, bool SELF, bool TAB>
__device__ __forceinline__ void inner_cplx(const WarpSmemCplx& sm, const double2* __restrict__ tab,
                                           int cnt, int j0, double kappa,
                                           const double (&xi)[R], const double (&yi)[R],
                                           const double (&zi)[R], const int (&rowi)[R],
                                           double2 (&au)[R], double2 (&ah)[R]) {
#pragma unroll kK2cUnroll
  for (int jj = 0; jj < cnt; ++jj) {
    const double2 xy = sm.xy[jj];
    const double zz = sm.z[jj];
    const double2 wa = sm.a[jj];
    const double2 wh = H ? sm.h[jj] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = xi[r] - xy.x, dy = yi[r] - xy.y, dz = zi[r] - zz;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double y = rsqrt_fp64(r2);
      double gr, gi;
      if constexpr (TAB) {
        sincos_tab_scaled(tab, KR_ARG(kappa, r2, y), y, &gr, &gi);
      } else {  // arguments beyond the table's exact reduction range
        double s, c;
        sincos_fast(kappa * (r2 * y), &s, &c);
        gr = c * y;
        gi = s * y;
      }
      if (SELF && rowi[r] == j0 + jj) {
        gr = 0.0;
        gi = 0.0;
      }
      au[r].x = fma(gr, wa.x, fma(-gi, wa.y, au[r].x));
      au[r].y = fma(gr, wa.y, fma(gi, wa.x, au[r].y));
      if (H) {
        ah[r].x = fma(gr, wh.x, fma(-gi, wh.y, ah[r].x));
        ah[r].y = fma(gr, wh.y, fma(gi, wh.x, ah[r].y));
      }
    }
  }
}

// kSYM for the complex kernel: as sym_chunk (rotation, fixed order) with
// complex row and column accumulators; columns past the source box are given
// G = 0 explicitly (a far-away padding point would make exp(i kappa r) NaN).
template <int R, bool H, bool TAB, bool CHAIN>
__device__ __forceinline__ void sym_chunk_cplx(const WarpSmemCplx& sm, const double2* __restrict__ tab,
                                               int j0, int n_c, int k_c, double kappa,
                                               const double (&xi)[R], const double (&yi)[R],
                                               const double (&zi)[R], const double2 (&qr)[R],
                                               const double2 (&qhr)[R], double2 (&au)[R],
                                               double2 (&ah)[R], double2* __restrict__ st_u,
                                               double2* __restrict__ st_h, int lane) {
  double2 cp = make_double2(0.0, 0.0), ch = make_double2(0.0, 0.0);
  if (!CHAIN && sm.tile > 0) {  // merged task: as sym_chunk
    const int col = j0 + lane;
    if (col < n_c) cp = st_u[col];
    if (H && col < k_c) ch = st_h[col];
  }
  const int from = (lane + 1) & 31;
  const int cnt = n_c - j0;  // valid columns of this chunk (may exceed 32)
#pragma unroll kSymCplxUnroll
  for (int s = 0; s < 32; ++s) {
    const int jc = (lane + s) & 31;
    const double2 xy = sm.xy[jc];
    const double zz = sm.z[jc];
    const double2 wa = sm.a[jc];
    const double2 wh = H ? sm.h[jc] : make_double2(0.0, 0.0);
    const bool valid = jc < cnt;
    double2 cs = make_double2(0.0, 0.0), hs = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double dx = xi[r] - xy.x, dy = yi[r] - xy.y, dz = zi[r] - zz;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double y = rsqrt_fp64(r2);
      double gr, gi;
      if constexpr (TAB) {
        sincos_tab_scaled(tab, KR_ARG(kappa, r2, y), y, &gr, &gi);
      } else {
        double sn, c;
        sincos_fast(kappa * (r2 * y), &sn, &c);
        gr = c * y;
        gi = sn * y;
      }
      gr = valid ? gr : 0.0;
      gi = valid ? gi : 0.0;
      au[r].x = fma(gr, wa.x, fma(-gi, wa.y, au[r].x));
      au[r].y = fma(gr, wa.y, fma(gi, wa.x, au[r].y));
      cs.x = fma(gr, qr[r].x, fma(-gi, qr[r].y, cs.x));
      cs.y = fma(gr, qr[r].y, fma(gi, qr[r].x, cs.y));
      if (H) {
        ah[r].x = fma(gr, wh.x, fma(-gi, wh.y, ah[r].x));
        ah[r].y = fma(gr, wh.y, fma(gi, wh.x, ah[r].y));
        hs.x = fma(gr, qhr[r].x, fma(-gi, qhr[r].y, hs.x));
        hs.y = fma(gr, qhr[r].y, fma(gi, qhr[r].x, hs.y));
      }
    }
    cp.x = __shfl_sync(kFull, cp.x + cs.x, from);
    cp.y = __shfl_sync(kFull, cp.y + cs.y, from);
    if (H) {
      ch.x = __shfl_sync(kFull, ch.x + hs.x, from);
      ch.y = __shfl_sync(kFull, ch.y + hs.y, from);
    }
  }
  chain_store<double2, H, CHAIN>(st_u, st_h, cp, ch, j0 + lane, n_c, k_c, &sm.fbase, &sm.tile, j0,
                                 lane);
}

template <int R, bool TAB, bool CHAIN>
__device__ __forceinline__ void task_cplx(const K2Args& a, const Task& t, WarpSmemCplx& sm,
                                          const double2* tab, int lane) {
  const int row0 = sm.row0;
  const double2* Q = reinterpret_cast<const double2*>(a.Q);
  const double2* QH = reinterpret_cast<const double2*>(a.QH);
  const BoxRec tb = a.box[t.box];
  double xi[R], yi[R], zi[R];
  double2 au[R], ah[R], qr[R], qhr[R];
  int rowi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = row0 + r * 32 + lane;
    rowi[r] = row;
    const bool valid = row < row0 + sm.nrows;
    const int64_t s = tb.slot + (valid ? row : row0);
    xi[r] = a.X[s];
    yi[r] = a.Y[s];
    zi[r] = a.Z[s];
    au[r] = make_double2(0.0, 0.0);
    ah[r] = make_double2(0.0, 0.0);
    qr[r] = valid ? Q[s] : make_double2(0.0, 0.0);  // row charges feed kSYM column sums
    qhr[r] = (valid && row < tb.k) ? QH[tb.skel + row] : make_double2(0.0, 0.0);
  }
  const EntryRange er = a.er[t.box];
  const bool skel_rows = row0 < tb.k;
  // one staged vector per pair for every row tile: chained or merged layout
  const bool pair_stage = CHAIN || t.nrows > sm.nrows;
  double2* St = reinterpret_cast<double2*>(a.St);
  int64_t stage = t.stage;
  for (int e = 0; e < er.count; ++e) {
    const int32_t code = a.ent[er.begin + e];
    const int32_t c = code >> kModeBits;
    const int mode = code & kModeMask;
    const BoxRec sb = a.box[c];
    if (mode == kSYM) {
      double2* st_u = St + stage;
      double2* st_h = st_u + sb.n;
      if (CHAIN && lane == 0) {
        sm.fbase = a.sflag + (stage >> 5);
        sm.tile = t.tile;
      }
      for (int j0 = 0; j0 < sb.n; j0 += 32) {
        const int j = j0 + lane;
        if (j < sb.n) {
          const int64_t s = sb.slot + j;
          sm.xy[lane] = make_double2(a.X[s], a.Y[s]);
          sm.z[lane] = a.Z[s];
          sm.a[lane] = Q[s];
          sm.h[lane] = j < sb.k ? QH[sb.skel + j] : make_double2(0.0, 0.0);
        } else {  // zero weights; G is zeroed for these columns
          sm.xy[lane] = make_double2(0.0, 0.0);
          sm.z[lane] = 0.0;
          sm.a[lane] = make_double2(0.0, 0.0);
          sm.h[lane] = make_double2(0.0, 0.0);
        }
        __syncwarp();
        if (skel_rows && j0 < sb.k)
          sym_chunk_cplx<R, true, TAB, CHAIN>(sm, tab, j0, sb.n, sb.k, a.kappa, xi, yi, zi, qr, qhr, au,
                                       ah, st_u, st_h, lane);
        else
          sym_chunk_cplx<R, false, TAB, CHAIN>(sm, tab, j0, sb.n, sb.k, a.kappa, xi, yi, zi, qr, qhr, au,
                                        ah, st_u, st_h, lane);
        __syncwarp();
      }
      stage += (sb.n + (((pair_stage ? tb.k > 0 : skel_rows) && sb.k > 0) ? sb.k : 0) + 31) &
               ~(int64_t)31;
      continue;
    }
    const bool self = c == t.box;
    for (int j0 = 0; j0 < sb.n; j0 += 32) {
      const int j = j0 + lane;
      if (j < sb.n) {
        const int64_t s = sb.slot + j;
        const double2 q = Q[s];
        const double2 qh = j < sb.k ? QH[sb.skel + j] : make_double2(0.0, 0.0);
        double2 wa = q, wh = make_double2(0.0, 0.0);
        if (mode == kIFO) wh = qh;
        else if (mode == kIFS) wh = q;
        else if (mode == kTFO) wa = make_double2(q.x - qh.x, q.y - qh.y);
        sm.xy[lane] = make_double2(a.X[s], a.Y[s]);
        sm.z[lane] = a.Z[s];
        sm.a[lane] = wa;
        sm.h[lane] = wh;
      }
      __syncwarp();
      const int cnt = min(32, sb.n - j0);
      const bool need_h = skel_rows && (mode == kIFS || (mode == kIFO && j0 < sb.k));
      if (self) {
        if (need_h) inner_cplx<R, true, true, TAB>(sm, tab, cnt, j0, a.kappa, xi, yi, zi, rowi, au, ah);
        else inner_cplx<R, false, true, TAB>(sm, tab, cnt, j0, a.kappa, xi, yi, zi, rowi, au, ah);
      } else {
        if (need_h) inner_cplx<R, true, false, TAB>(sm, tab, cnt, j0, a.kappa, xi, yi, zi, rowi, au, ah);
        else inner_cplx<R, false, false, TAB>(sm, tab, cnt, j0, a.kappa, xi, yi, zi, rowi, au, ah);
      }
      __syncwarp();
    }
  }
  double2* U = reinterpret_cast<double2*>(a.U);
  double2* UH = reinterpret_cast<double2*>(a.UH);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = rowi[r];
    if (row >= sm.row0 + sm.nrows) continue;
    const bool skel_row = row < tb.k;
    if (!isfinite(au[r].x) || !isfinite(au[r].y) ||
        (skel_row && (!isfinite(ah[r].x) || !isfinite(ah[r].y))))
      verify_row(a, t.box, row, 3);
    U[tb.slot + row] = make_double2(au[r].x * 0.25, au[r].y * 0.25);
    if (skel_row) UH[tb.skel + row] = make_double2(-ah[r].x * 0.25, -ah[r].y * 0.25);
  }
}

#ifndef SFMM_K2C_MIN_BLOCKS
#define SFMM_K2C_MIN_BLOCKS 3
#endif
template <bool TAB, bool CHAIN>
__global__ void __launch_bounds__(kThreads, SFMM_K2C_MIN_BLOCKS) k2_translate_cplx(K2Args a) {
  __shared__ WarpSmemCplx smem[kWarps];
  __shared__ double2 tab[kSinCosTab];
  if (TAB)
    for (int i = threadIdx.x; i < kSinCosTab; i += blockDim.x) tab[i] = a.tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  WarpSmemCplx& sm = smem[threadIdx.x >> 5];
  if (lane == 0) sm.pend_t = -1;
  for (;;) {
    // the next tile: a merged task's next one, else a new task (as the real K2)
    int t = 0;
    if (lane == 0) {
      int r0 = 0;
      if (sm.pend_t >= 0) {
        t = sm.pend_t;
        r0 = sm.pend_r0;
      } else {
        t = atomicAdd(a.counter, 1);
      }
      sm.pend_t = -1;
      if (t < a.n_tasks) {
        constexpr int kTile = 32 * SFMM_K2C_MAX_R;
        const int nr = a.tasks[t].nrows;
        sm.row0 = a.tasks[t].row0 + r0;
        sm.nrows = min(kTile, nr - r0);
        if (!CHAIN) sm.tile = r0 / kTile;
        if (r0 + kTile < nr) {
          sm.pend_t = t;
          sm.pend_r0 = r0 + kTile;
        }
      }
    }
    t = __shfl_sync(kFull, t, 0);
    if (t >= a.n_tasks) return;
    const Task task = a.tasks[t];
    switch ((sm.nrows + 31) >> 5) {
      case 1: task_cplx<1, TAB, CHAIN>(a, task, sm, tab, lane); break;
#if SFMM_K2C_MAX_R >= 3
      case 2: task_cplx<2, TAB, CHAIN>(a, task, sm, tab, lane); break;
#endif
#if SFMM_K2C_MAX_R >= 4
      case 3: task_cplx<3, TAB, CHAIN>(a, task, sm, tab, lane); break;
#endif
      default: task_cplx<SFMM_K2C_MAX_R, TAB, CHAIN>(a, task, sm, tab, lane); break;
    }
    __syncwarp();
  }
}

// K2b: adds the staged kSYM column sums to their receiving boxes, summing the
// contributions in the (source box, row tile) order fixed at plan time.
__global__ void __launch_bounds__(256) k2b_reduce(const BoxRec* __restrict__ box,
                                                  const int32_t* __restrict__ recv_box,
                                                  const int64_t* __restrict__ recv_off,
                                                  const int64_t* __restrict__ recv_u,
                                                  const int64_t* __restrict__ recv_h,
                                                  const double* __restrict__ St,
                                                  double* __restrict__ U,
                                                  double* __restrict__ UH, double scale) {
  const BoxRec br = box[recv_box[blockIdx.x]];
  const int64_t e0 = recv_off[blockIdx.x], e1 = recv_off[blockIdx.x + 1];
  // the sums run in the fixed e order (deterministic); unrolling lets the
  // independent loads of several staged vectors be in flight at once
  for (int i = threadIdx.x; i < br.n; i += blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int64_t e = e0; e < e1; ++e) s += __ldg(St + recv_u[e] + i);
    U[br.slot + i] += scale * s;
    if (i < br.k) {
      double h = 0.0;
#pragma unroll 8
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t o = recv_h[e];
        h += o >= 0 ? __ldg(St + o + i) : 0.0;
      }
      UH[br.skel + i] -= scale * h;
    }
  }
}

__global__ void __launch_bounds__(256) k2b_reduce_cplx(const BoxRec* __restrict__ box,
                                                       const int32_t* __restrict__ recv_box,
                                                       const int64_t* __restrict__ recv_off,
                                                       const int64_t* __restrict__ recv_u,
                                                       const int64_t* __restrict__ recv_h,
                                                       const double2* __restrict__ St,
                                                       double2* __restrict__ U,
                                                       double2* __restrict__ UH, double scale) {
  const BoxRec br = box[recv_box[blockIdx.x]];
  const int64_t e0 = recv_off[blockIdx.x], e1 = recv_off[blockIdx.x + 1];
  for (int i = threadIdx.x; i < br.n; i += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int64_t e = e0; e < e1; ++e) {
      const double2 v = __ldg(St + recv_u[e] + i);
      s.x += v.x;
      s.y += v.y;
    }
    const double2 u = U[br.slot + i];
    U[br.slot + i] = make_double2(u.x + scale * s.x, u.y + scale * s.y);
    if (i < br.k) {
      double2 h = make_double2(0.0, 0.0);
#pragma unroll 4
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t o = recv_h[e];
        if (o >= 0) {
          const double2 v = __ldg(St + o + i);
          h.x += v.x;
          h.y += v.y;
        }
      }
      const double2 uh = UH[br.skel + i];
      UH[br.skel + i] = make_double2(uh.x - scale * h.x, uh.y - scale * h.y);
    }
  }
}

}  // namespace

int configure_translate(DevPlan& p, int device) {
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return -1;
  cudaError_t e;
  if (p.kernel == SFMM_HELMHOLTZ3D)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_translate_cplx<true, false>,
                                                      kThreads, 0);
  else if (p.kernel == SFMM_LAPLACE3D)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k2_real_kernel<GenLaplace3d>(p.k2_r1, p.sym_chain, p.k2_merged), kThreads, 0);
  else
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k2_real_kernel<GenLaplace2d>(p.k2_r1, p.sym_chain, p.k2_merged), kThreads, 0);
  if (e != cudaSuccess) return -1;
  if (per_sm < 1) per_sm = 1;
  p.k2_grid = sms * per_sm;
  return 0;
}

void launch_translate(const DevPlan& p, DevState& s, cudaStream_t st, TranslatePart part,
                      bool reduce) {
  const size_t sw = p.cplx ? 16 : 8;
  if (part != kBoundaryTasks) {
    // boxes whose every entry cancels own no task: their U/UH stay zero
    cudaMemsetAsync(s.U, 0, (size_t)p.n_slots * sw, st);
    cudaMemsetAsync(s.UH, 0, (size_t)p.n_skel * sw, st);
    // chained kSYM column sums start from "no tile has added"
    if (p.stage_size > 0)
      cudaMemsetAsync(p.stage_flags, 0, sizeof(unsigned) * (size_t)(p.stage_size >> 5), st);
  }
  int64_t t0 = 0, t1 = p.n_tasks;
  int* counter = p.counter;
  if (part == kInteriorTasks) t1 = p.n_interior;
  if (part == kBoundaryTasks) {
    t0 = p.n_interior;
    counter = p.counter + 1;
  }
  if (t1 > t0) {
    K2Args a;
    a.box = p.box;
    a.er = p.ent_range;
    a.ent = p.entries;
    a.tasks = p.tasks + t0;
    a.n_tasks = t1 - t0;
    a.X = p.X;
    a.Y = p.Y;
    a.Z = p.Z;
    a.sid = p.slot_id;
    a.Q = s.Q;
    a.QH = s.QH;
    a.U = s.U;
    a.UH = s.UH;
    a.counter = counter;
    a.err = p.err_flag;
    a.kappa = p.kappa;
    a.tab = p.sc_tab;
    a.ltab = p.log_tab;
    a.St = p.stage;
    a.sflag = p.stage_flags;
    cudaMemsetAsync(counter, 0, sizeof(int), st);
    const int grid = (int)std::min<int64_t>(p.k2_grid, (t1 - t0 + kWarps - 1) / kWarps);
    if (p.kernel == SFMM_HELMHOLTZ3D) {
      auto kc = p.sc_tab_ok ? (p.sym_chain ? k2_translate_cplx<true, true>
                                           : k2_translate_cplx<true, false>)
                            : (p.sym_chain ? k2_translate_cplx<false, true>
                                           : k2_translate_cplx<false, false>);
      kc<<<grid, kThreads, 0, st>>>(a);
    } else if (p.kernel == SFMM_LAPLACE3D) {
      k2_real_kernel<GenLaplace3d>(p.k2_r1, p.sym_chain, p.k2_merged)<<<grid, kThreads, 0, st>>>(a);
    } else {
      k2_real_kernel<GenLaplace2d>(p.k2_r1, p.sym_chain, p.k2_merged)<<<grid, kThreads, 0, st>>>(a);
    }
  }
  if (part != kInteriorTasks && reduce) launch_stage_reduce(p, s, st);
}

void launch_stage_reduce(const DevPlan& p, DevState& s, cudaStream_t st) {
  if (p.n_recv > 0 && p.cplx) {
    k2b_reduce_cplx<<<(unsigned)p.n_recv, 256, 0, st>>>(
        p.box, p.recv_box, p.recv_off, p.recv_u, p.recv_h, reinterpret_cast<const double2*>(p.stage),
        reinterpret_cast<double2*>(s.U), reinterpret_cast<double2*>(s.UH), 0.25);
  } else if (p.n_recv > 0) {
    const double scale = p.kernel == SFMM_LAPLACE3D ? GenLaplace3d::kScale : GenLaplace2d::kScale;
    k2b_reduce<<<(unsigned)p.n_recv, 256, 0, st>>>(p.box, p.recv_box, p.recv_off, p.recv_u,
                                                   p.recv_h, p.stage, s.U, s.UH, scale);
  }
}

}  // namespace sfmm_gpu
