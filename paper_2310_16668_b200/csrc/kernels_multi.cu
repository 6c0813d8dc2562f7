// Multi-right-hand-side apply (nrhs > 1): K0m, K1m, K2m, K3m, K4m.
//
// The reference applies one right-hand side per call (apply.hpp:91-94); a
// user with 16 charge vectors runs fmm_apply 16 times and regenerates every
// kernel entry 16 times.  Here the right-hand sides go through the tree
// together, 16 at a time, so each G(x_i, x_j) is generated once and applied to
// all of them: the translation step becomes a generated-matrix x (n_c x 16)
// product issued on the FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA).
//
// K2m task = 64 target rows of one box on one CTA: 4 warps x two 8-row DMMA
// tiles, sharing each staged 16-source chunk (B operands pre-arranged in
// fragment order; the next chunk's loads are in flight during the compute).
// Per k-step (4 sources) every lane generates the one G entry its A-fragment
// holds (row = lane/4, source = lane%4) -- one pair per lane, no shuffles --
// and the warp issues 6 DMMAs (complex) or 2 (real) per row tile.  Complex products use
// the 3-multiplication form T1 = Gr Ar, T2 = Gi Ai, T3 = (Gr + Gi)(Ar + Ai),
// Re U = T1 - T2, Im U = T3 - T1 - T2 (25 % fewer DMMAs than the 4-product
// form; error bound eps * sum |G||A| like it).  On B200 DMMA shares the FP64 datapath with DFMA (both
// measured at 37 TFLOP/s, see profiles/), so the gain over scalar code is
// issue slots and registers, not peak.
#include <math.h>

#include <algorithm>

#include "fastmath.cuh"
#include "launch.h"

namespace sfmm_gpu {
namespace {

constexpr int kMWarps = 4;
constexpr int kMThreads = 32 * kMWarps;
constexpr int kChunk = kChunkM;  // sources staged per chunk (4 k-steps of 4)
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
  const double2* tab;  // (cos, sin)(k pi/128), Helmholtz only
  const double* ltab;  // log table, Laplace 2D only
  const int32_t* soff; // symmetric u pass: per entry, first staged point of a kSYM entry
  double* stage;       // symmetric u pass: staged column sums [point][kNRHS] (pre-scaled)
  unsigned* sflag;     // symmetric u pass: per staged chunk, warps of the tiles that have added
};

// A task's whole entry list (source box records, codes, staged offsets) is
// held in shared memory, so the chunk iterator never touches global memory;
// plans with a longer list take the column loop instead (configure_multi).
constexpr int kMEntCap = 256;

__device__ __forceinline__ unsigned ld_acquire_flag(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

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

// One staged 16-source chunk, shared by the CTA's 4 warps.  The B operands are
// stored in DMMA fragment order ([k-step][B1|B2][n-block][lane]) so each lane
// loads its fragment with one conflict-free 8-byte LDS.
template <bool CPLX>
struct ChunkM {
  static constexpr int NB = 2;             // 8-column rhs blocks
  static constexpr int NP = CPLX ? 3 : 1;  // B = Ar, Ai, Ar + Ai (complex) or A
  double x[kChunk], y[kChunk], z[kChunk];
  double w[4][NP][NB][32];  // the pass's weights (u pass: a, uhat pass: h)
};

// Symmetric u pass (kSYM entries): the CTA's generated 64 x 16 block of a
// chunk and the task's own charges (64 rows x kNRHS), both [row][16] in
// shared memory with the 16-column index XOR-swizzled by the row so the
// transposed fragment loads (4 rows x 8 columns per k-step) and the
// generation stores are (nearly) conflict-free.
template <bool CPLX>
__device__ __forceinline__ int swz(int row, int col) {
  return col ^ ((row & 3) << (CPLX ? 1 : 2));
}

// Raw per-thread staging payload of one chunk (registers), so the next chunk's
// global loads are in flight while the current one is computed.
template <bool CPLX>
struct StageRegs {
  static constexpr int SW = CPLX ? 2 : 1;
  static constexpr int ITEMS = kChunk * kNRHS / kMThreads;  // (source, rhs) per thread
  // the pass's weight (u pass: q; uhat pass: qhat for ifo, q for ifs) and,
  // for plans with tfo entries, qhat for the u pass's tfo weight q - qhat
  double w[ITEMS][SW], w2[ITEMS][SW];
  double cx, cy, cz;
};

struct ChunkPos {
  int e, j0;  // entry index, first source of the chunk
};

// KER: 0 laplace2d, 1 laplace3d, 3 helmholtz3d
// HPASS: false = the u pass over every task (U = sum G a); true = the uhat
// pass over the tasks owning skeleton rows (UH = -sum G h), visiting only the
// chunks that carry an h weight (ifs entries, and the skeleton sources of ifo
// entries: ~1/8 of the columns).  Round 1 accumulated both in one variant;
// its 96 accumulator registers spilled (168 registers, ~1.3e9 local-memory
// instructions per config-4 apply, 44 % of K2m's time for ~1/5 of the rows).
// Two passes with one accumulator set each regenerate G for the few h chunks
// instead.
// TAB: Helmholtz arguments within the sincos table's range (sincos_fast otherwise).
#ifndef SFMM_K2M_MIN_BLOCKS
#define SFMM_K2M_MIN_BLOCKS 4  // measured: 4 > 3 on config 4
#endif
// TFO: the plan has tfo entries (u pass needs q and qhat of those sources).
// SYM: the u pass over the folded lists (HostPlan::multi_sym): a kSYM chunk's
// generated block is also applied transposed to the task's charges -- warp w
// takes sources 8(w&1).. and rhs block w>>1 over all the task's rows -- and
// the column sums go to the staging buffer (K2bm adds them).  Its shared
// memory (two block buffers + the charges) allows 3 CTAs per SM (complex).
#ifndef SFMM_K2M_SYM_MIN_BLOCKS
#define SFMM_K2M_SYM_MIN_BLOCKS 3
#endif
template <int KER, bool HPASS, bool TAB, bool TFO, bool SYM>
__global__ void __launch_bounds__(kMThreads, SYM ? (KER == SFMM_HELMHOLTZ3D ? SFMM_K2M_SYM_MIN_BLOCKS : 4)
                                                 : SFMM_K2M_MIN_BLOCKS)
    k2m_translate(K2MArgs a) {
  static_assert(!(SYM && HPASS), "the symmetric fold is a u-pass variant");
  constexpr bool CPLX = KER == SFMM_HELMHOLTZ3D;
  constexpr int SW = CPLX ? 2 : 1;
  constexpr int NB = 2;             // rhs blocks of 8
  constexpr int NP = CPLX ? 3 : 1;  // real products per complex product (3M)
  constexpr int DIM = KER == SFMM_LAPLACE2D ? 2 : 3;
  constexpr int ITEMS = StageRegs<CPLX>::ITEMS;
  // two chunk buffers: the next chunk is stored while the current one is
  // read, so one barrier per chunk suffices
  __shared__ ChunkM<CPLX> chb[2];
  ChunkM<CPLX>* chp = &chb[0];
  __shared__ int s_task;
  // the task's entry list (codes and source box records), read once per task:
  // the chunk iterator then runs from shared memory instead of two dependent
  // global loads per chunk on the critical path
  __shared__ int32_t s_code[kMEntCap];
  __shared__ BoxRec s_sb[kMEntCap];
  __shared__ int32_t s_soff[SYM ? kMEntCap : 1];
  // SYM (dynamic shared memory, sym_smem_bytes): generated blocks of the
  // current / previous kSYM chunk and the task's charges, [row][16 columns]
  // of scalars (complex: interleaved)
  extern __shared__ __align__(16) double k2m_dyn[];
  using GRow = double[kChunk * SW];
  GRow* gts0 = reinterpret_cast<GRow*>(k2m_dyn);
  GRow* qbs = gts0 + 2 * kMultiRows;
  __shared__ double2 tab[CPLX ? kSinCosTab : 1];
  __shared__ __align__(16) double ltab[KER == SFMM_LAPLACE2D ? kLogTabLen : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (CPLX && TAB)
    for (int i = tid; i < kSinCosTab; i += blockDim.x) tab[i] = a.tab[i];
  if (KER == SFMM_LAPLACE2D)
    for (int i = tid; i < kLogTabLen; i += blockDim.x) ltab[i] = a.ltab[i];
  const uint32_t lts = log_tab_addr(ltab);
  const int rq = lane >> 2, kq = lane & 3;  // A-fragment row / k index of this lane
  for (;;) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(a.counter, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.n_tasks) return;
    const Task task = a.tasks[t];
    const BoxRec tb = a.box[task.box];
    const EntryRange er = a.er[task.box];
    for (int i = tid; i < er.count; i += kMThreads) {  // er.count <= kMEntCap (configure_multi)
      const int32_t code = a.ent[er.begin + i];
      s_code[i] = code;
      s_sb[i] = a.box[code >> kModeBits];
      if (SYM) s_soff[i] = a.soff[er.begin + i];
    }
    __syncthreads();
    if constexpr (SYM) {  // the task's charges (zero past its rows); ordered by the barrier before the loop
      for (int v = tid; v < kMultiRows * kNRHS; v += kMThreads) {
        const int row = v / kNRHS, r = v % kNRHS;
        const int cs = swz<CPLX>(row, r) * SW;
        if (row < task.nrows) {
          const double* qp = a.Q + ((tb.slot + task.row0 + row) * kNRHS + r) * SW;
#pragma unroll
          for (int c = 0; c < SW; ++c) qbs[row][cs + c] = qp[c];
        } else {
#pragma unroll
          for (int c = 0; c < SW; ++c) qbs[row][cs + c] = 0.0;
        }
      }
    }
    auto ent_code = [&](int e) -> int32_t { return s_code[e]; };
    auto ent_soff = [&](int e) -> int32_t { return s_soff[e]; };
    auto ent_box = [&](int e) -> BoxRec { return s_sb[e]; };
    const int wrow0 = task.row0 + 16 * warp;  // this warp's 16 rows
    // the uhat pass needs the skeleton rows only: warps past them skip the chunk
    // work entirely (a box's last skeleton tile is often mostly redundant rows)
    const int rend = task.row0 + (HPASS ? min(task.nrows, tb.k - task.row0) : task.nrows);
    double xr[2], yr[2], zr[2];
    int rowi[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = wrow0 + mt * 8 + rq;
      rowi[mt] = row;
      const int64_t s = tb.slot + (row < rend ? row : task.row0);
      xr[mt] = a.X[s];
      yr[mt] = a.Y[s];
      zr[mt] = DIM == 3 ? a.Z[s] : 0.0;
    }
    double C[2][NP][NB][2];  // u accumulators (HPASS: uhat)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) C[mt][pp][nb][0] = C[mt][pp][nb][1] = 0.0;

    // chunk iterator over (entry, first source), skipping empty source boxes;
    // the uhat pass visits only chunks with an h weight (ifs: every source;
    // ifo: the skeleton sources j < k_c)
    auto h_limit = [&](int e) -> int {
      const int32_t code = ent_code(e);
      const int mode = code & kModeMask;
      const BoxRec sb = ent_box(e);
      if (!HPASS) return sb.n;
      return mode == kIFS ? sb.n : (mode == kIFO ? sb.k : 0);
    };
    auto first_from = [&](int e) -> ChunkPos {
      for (; e < er.count; ++e)
        if (h_limit(e) > 0) return {e, 0};
      return {er.count, 0};
    };
    auto next_of = [&](ChunkPos p) -> ChunkPos {
      if (p.j0 + kChunk < h_limit(p.e)) return {p.e, p.j0 + kChunk};
      return first_from(p.e + 1);
    };
    // global loads of one chunk into registers (raw q and qhat)
    // Item it of this thread is (source jj, rhs r) with the warp's 32 lanes
    // covering one (k-step, rhs half) block in fragment-lane order, so the
    // fragment stores below are conflict-free.
    auto item = [&](int it, int& jj, int& r) {
      const int g = warp + kMWarps * it;  // 0..7: (k-step, rhs half)
      jj = 4 * (g >> 1) + (lane & 3);
      r = 8 * (g & 1) + (lane >> 2);
    };
    auto load = [&](ChunkPos p, StageRegs<CPLX>& R) {
      const BoxRec sb = ent_box(p.e);
      const int mode = ent_code(p.e) & kModeMask;
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        int jj, r;
        item(it, jj, r);
        const int j = p.j0 + jj;
#pragma unroll
        for (int c = 0; c < SW; ++c) R.w[it][c] = R.w2[it][c] = 0.0;
        if (j < sb.n) {
          const double* qp = a.Q + ((sb.slot + j) * kNRHS + r) * SW;
          const double* hp = a.QH + ((sb.skel + j) * kNRHS + r) * SW;
          if (HPASS) {
            if (mode == kIFS) {
#pragma unroll
              for (int c = 0; c < SW; ++c) R.w[it][c] = qp[c];
            } else if (j < sb.k) {  // ifo: qhat on the skeleton sources
#pragma unroll
              for (int c = 0; c < SW; ++c) R.w[it][c] = hp[c];
            }
          } else {
#pragma unroll
            for (int c = 0; c < SW; ++c) R.w[it][c] = qp[c];
            if (TFO && mode == kTFO && j < sb.k) {
#pragma unroll
              for (int c = 0; c < SW; ++c) R.w2[it][c] = hp[c];
            }
          }
        }
      }
      if (tid < kChunk) {
        const int j = p.j0 + tid;
        if (j < sb.n) {
          const int64_t s = sb.slot + j;
          R.cx = a.X[s];
          R.cy = a.Y[s];
          R.cz = DIM == 3 ? a.Z[s] : 0.0;
        } else {  // far away, zero weight (moderate: sincos stays on its fast path)
          R.cx = R.cy = R.cz = 1e3;
        }
      }
    };
    // per-mode weights, scattered into fragment order (the u pass stores the
    // a weights, the uhat pass -- need_h -- the h weights)
    auto store = [&](ChunkPos p, const StageRegs<CPLX>& R, bool need_h) {
      const int mode = ent_code(p.e) & kModeMask;
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        int jj, r;
        item(it, jj, r);
        const int ks = jj >> 2, fl = 4 * (r & 7) + (jj & 3);  // fragment lane (== lane)
        double wa[SW], wh[SW];
#pragma unroll
        for (int c = 0; c < SW; ++c) {
          wa[c] = R.w[it][c];
          if (TFO && !HPASS && mode == kTFO) wa[c] = R.w[it][c] - R.w2[it][c];
          wh[c] = R.w[it][c];
        }
        const double w0 = need_h ? wh[0] : wa[0], w1 = need_h ? wh[SW - 1] : wa[SW - 1];
        const int nb = r >> 3;
        chp->w[ks][0][nb][fl] = w0;
        if (CPLX) {
          chp->w[ks][NP - 2][nb][fl] = w1;
          chp->w[ks][NP - 1][nb][fl] = w0 + w1;
        }
      }
      if (tid < kChunk) {
        chp->x[tid] = R.cx;
        chp->y[tid] = R.cy;
        chp->z[tid] = R.cz;
      }
    };
    ChunkPos cur = first_from(0);
    StageRegs<CPLX> R;
    int buf = 0;
    if (cur.e < er.count) {
      load(cur, R);
      chp = &chb[0];
      store(cur, R, HPASS);
    }
    __syncthreads();
    ChunkPos nxt = cur.e < er.count ? next_of(cur) : cur;
    if (nxt.e < er.count) load(nxt, R);  // in flight during the compute below
    // SYM: the kSYM chunk whose transposed product is still due (it runs one
    // iteration late, reading the block buffer the previous iteration wrote)
    ChunkPos prev{er.count, 0};
    auto is_sym = [&](const ChunkPos& p) {
      return SYM && p.e < er.count && (ent_code(p.e) & kModeMask) == kSYM;
    };
    while (cur.e < er.count || is_sym(prev)) {
      chp = &chb[buf];
      const bool live = !SYM || cur.e < er.count;  // (without SYM the loop runs live chunks only)
      const int32_t code = live ? ent_code(cur.e) : 0;
      const bool self = live && (code >> kModeBits) == task.box;
      const bool csym = SYM && live && (code & kModeMask) == kSYM;
      const int j0 = cur.j0;
      // sources of this chunk past the box end are padding: their G is masked
      // below (never trusted to vanish through the zero weight: a target may
      // sit exactly at the padding coordinate)
      const int n_valid = live ? ent_box(cur.e).n - j0 : 0;
      if (live && wrow0 < rend) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int js = 4 * ks + kq;  // this lane's source within the chunk
          double gr[2], gi[2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const double dx = xr[mt] - chp->x[js], dy = yr[mt] - chp->y[js];
            double r2 = fma(dy, dy, dx * dx);
            if (DIM == 3) {
              const double dz = zr[mt] - chp->z[js];
              r2 = fma(dz, dz, r2);
            }
            if (KER == SFMM_LAPLACE2D) {
              gr[mt] = log_tab(lts, r2);
              gi[mt] = 0.0;
            } else {
              const double yv = rsqrt_fp64m(r2);
              if (CPLX) {
                if constexpr (TAB) {
                  sincos_tab_scaled(tab, KR_ARG(a.kappa, r2, yv), yv, &gr[mt], &gi[mt]);
                } else {
                  double sn, cs;
                  sincos_fast(a.kappa * (r2 * yv), &sn, &cs);
                  gr[mt] = cs * yv;
                  gi[mt] = sn * yv;
                }
              } else {
                gr[mt] = yv;
                gi[mt] = 0.0;
              }
            }
            if ((self && rowi[mt] == j0 + js) || js >= n_valid) gr[mt] = gi[mt] = 0.0;
            if constexpr (SYM) if (csym) {  // the block, for the transposed product one iteration later
              const int rl = 16 * warp + 8 * mt + rq;
              double* gp = &gts0[buf * kMultiRows + rl][swz<CPLX>(rl, js) * SW];
              gp[0] = gr[mt];
              if (CPLX) gp[SW - 1] = gi[mt];
            }
          }
          // A operands of the NP real products: Gr (, Gi, Gr + Gi)
          double g[NP][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            g[0][mt] = gr[mt];
            if (CPLX) {
              g[NP - 2][mt] = gi[mt];
              g[NP - 1][mt] = gr[mt] + gi[mt];
            }
          }
#pragma unroll
          for (int pp = 0; pp < NP; ++pp)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              const double bv = chp->w[ks][pp][nb][lane];
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) dmma(C[mt][pp][nb][0], C[mt][pp][nb][1], g[pp][mt], bv);
            }
        }
      }
      if constexpr (SYM) if (is_sym(prev)) {
        // column sums of the previous kSYM chunk: D (8 sources x 8 rhs) +=
        // G^T (8 sources x 4 rows) * q_b (4 rows x 8 rhs) over the task's rows
        const int ms = 8 * (warp & 1), nbs = 8 * (warp >> 1);
        constexpr int NACC = CPLX ? 2 : 4;  // independent accumulator chains
        double D[NACC][NP][2];
#pragma unroll
        for (int u = 0; u < NACC; ++u)
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) D[u][pp][0] = D[u][pp][1] = 0.0;
        const int nks = (task.nrows + 3) >> 2;
        const GRow* gb = gts0 + (buf ^ 1) * kMultiRows;
        for (int k0 = 0; k0 < nks; k0 += NACC) {
#pragma unroll
          for (int u = 0; u < NACC; ++u) {
            if (k0 + u < nks) {
              const int row = 4 * (k0 + u) + kq;
              const double* gp = &gb[row][swz<CPLX>(row, ms + rq) * SW];
              const double* qp = &qbs[row][swz<CPLX>(row, nbs + rq) * SW];
              double ga[NP], qa[NP];
              ga[0] = gp[0];
              qa[0] = qp[0];
              if (CPLX) {
                ga[NP - 2] = gp[SW - 1];
                ga[NP - 1] = ga[0] + ga[NP - 2];
                qa[NP - 2] = qp[SW - 1];
                qa[NP - 1] = qa[0] + qa[NP - 2];
              }
#pragma unroll
              for (int pp = 0; pp < NP; ++pp) dmma(D[u][pp][0], D[u][pp][1], ga[pp], qa[pp]);
            }
          }
        }
        // the pair's staged vector is shared by b's row tiles: tile t adds to
        // what tiles 0..t-1 left (in tile order: deterministic), then counts
        // this warp into the chunk's flag (4 warps per tile)
        const int64_t cpt = task.stage + ent_soff(prev.e) + prev.j0;  // the chunk's first point
        unsigned* flag = a.sflag + cpt / kChunk;
        if (task.tile > 0) {
          if (lane == 0)
            while (ld_acquire_flag(flag) < (unsigned)(kMWarps * task.tile)) __nanosleep(64);
          __syncwarp();
        }
        const int j = prev.j0 + ms + rq;  // this lane's source (column of the block)
        if (j < ent_box(prev.e).n) {
          const double scale = CPLX ? 0.25 : (KER == SFMM_LAPLACE3D ? kInv4Pi : -kInv4Pi);
          double* out = a.stage + ((cpt + ms + rq) * kNRHS + nbs + 2 * kq) * SW;
          double o[2 * SW];
#pragma unroll
          for (int c = 0; c < 2 * SW; ++c) o[c] = task.tile > 0 ? __ldcg(out + c) : 0.0;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            double t[NP];
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
              t[pp] = D[0][pp][w];
#pragma unroll
              for (int u = 1; u < NACC; ++u) t[pp] += D[u][pp][w];
            }
            if (CPLX) {
              __stcg(out + 2 * w, o[2 * w] + (t[0] - t[NP - 2]) * scale);
              __stcg(out + 2 * w + 1, o[2 * w + 1] + (t[NP - 1] - t[0] - t[NP - 2]) * scale);
            } else {
              __stcg(out + w, o[w] + t[0] * scale);
            }
          }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(flag, 1u);
      }
      if (nxt.e < er.count) {  // the other buffer was last read before the previous barrier
        chp = &chb[buf ^ 1];
        store(nxt, R, HPASS);
      }
      __syncthreads();
      buf ^= 1;
      prev = cur;
      cur = nxt;
      if (cur.e < er.count) {
        nxt = next_of(cur);
        if (nxt.e < er.count) load(nxt, R);
      }
    }
    // epilogue: lane holds rows rq (+8) and rhs columns c0, c0+1, 8+c0, 9+c0
    const double scale = CPLX ? 0.25 : (KER == SFMM_LAPLACE3D ? kInv4Pi : -kInv4Pi);
    const int c0 = kq * 2;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = rowi[mt];
      if (row >= rend) continue;
      bool bad = false;
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          bad = bad || !isfinite(C[mt][pp][nb][0]) || !isfinite(C[mt][pp][nb][1]);
      if (bad) verify_row_m(a, task.box, row, DIM);
      if (HPASS && row >= tb.k) continue;  // uhat exists for skeleton rows only
      // u pass: U = scale * acc; uhat pass: UH = -scale * acc
      double* out = HPASS ? a.UH + (tb.skel + row) * (kNRHS * SW)
                          : a.U + (tb.slot + row) * (kNRHS * SW);
      const double sc = HPASS ? -scale : scale;
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // rhs block c0 + 8*half
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int rhs = c0 + 8 * half + w;
          if (CPLX) {
            const double t1 = C[mt][0][half][w], t2 = C[mt][NP - 2][half][w];
            out[2 * rhs] = (t1 - t2) * sc;
            out[2 * rhs + 1] = (C[mt][NP - 1][half][w] - t1 - t2) * sc;
          } else {
            out[rhs] = C[mt][0][half][w] * sc;
          }
        }
      }
    }
  }
}

// ---- tree passes for kNRHS right-hand sides ------------------------------

// K0m: Qm[slot][r] = q[orig + r*N] for r < nc, 0 for the padding columns.
template <class S>
__global__ void k0m_gather(const int32_t* __restrict__ slot, const int32_t* __restrict__ orig,
                           int64_t n_owned, int64_t N, int nc, const S* __restrict__ q,
                           S* __restrict__ Q) {
  const int64_t total = n_owned * kNRHS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kNRHS;
    const int r = (int)(i % kNRHS);
    S v{};
    if (r < nc) v = q[(int64_t)r * N + orig[t]];
    Q[(int64_t)slot[t] * kNRHS + r] = v;
  }
}

template <class S>
__global__ void k4m_scatter(const int32_t* __restrict__ slot, const int32_t* __restrict__ orig,
                            int64_t n_owned, int64_t N, int nc, const S* __restrict__ U,
                            S* __restrict__ u) {
  const int64_t total = n_owned * kNRHS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kNRHS;
    const int r = (int)(i % kNRHS);
    if (r < nc) u[(int64_t)r * N + orig[t]] = U[(int64_t)slot[t] * kNRHS + r];
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 t, double2 u) {  // conj(t) * u
  return make_double2(fma(t.x, u.x, t.y * u.y), fma(t.x, u.y, -t.y * u.x));
}

// ---- K1m / K3m: the interpolation operators applied to 16 right-hand sides
// at once, a (k x r) x (r x 16) product per box on the FP64 tensor cores
// (DMMA m8n8k4; complex via the 3-multiplication form as in K2m).  Each warp
// owns 16 rows (two 8-row tiles) x 16 right-hand sides (two 8-column blocks):
// A fragments come straight from T (each lane one element, rows of 4
// consecutive entries), B fragments from the right-hand-side block staged in
// shared memory, [row][16] with the column XOR-swizzled by the row so the
// fragment loads (4 rows x 8 columns) are conflict-free.
template <class S>
__device__ __forceinline__ int swz_m(int row, int col) {
  return col ^ ((row & 3) << (sizeof(S) == 16 ? 1 : 2));
}

// 3M split of a complex value into the A / B operands of the three products
__device__ __forceinline__ void parts3(double2 v, double (&o)[3]) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.x + v.y;
}
__device__ __forceinline__ void parts3(double v, double (&o)[1]) { o[0] = v; }

constexpr int kUpRowsM = kUpRows;  // K1m rows per CTA: 4 warps x 16
static_assert(kUpRowsM == 64, "K1m: four warps of 16 rows");

// K1m: qhat[i][.] = Q[i][.] + sum_j T[i,j] Q[k+j][.] for the item's 64
// skeleton rows; the q_R block is staged 64 sources at a time.
template <class S>
__global__ void __launch_bounds__(128) k1m_upward(const LevelItem* __restrict__ items,
                                                  const BoxRec* __restrict__ box,
                                                  const int64_t* __restrict__ T_off,
                                                  const S* __restrict__ T, S* __restrict__ Q,
                                                  S* __restrict__ QH,
                                                  const int32_t* __restrict__ up_dst) {
  constexpr bool CPLX = sizeof(S) == 16;
  constexpr int NP = CPLX ? 3 : 1;
  __shared__ S sq[64][kNRHS];
  const LevelItem it = items[blockIdx.x];
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rq = lane >> 2, kq = lane & 3;
  const S* Tb = T + T_off[it.box];
  double C[2][NP][2][2] = {};
  int rowi[2];
  for (int mt = 0; mt < 2; ++mt) rowi[mt] = it.first + 16 * warp + 8 * mt + rq;
  for (int j0 = 0; j0 < r; j0 += 64) {
    __syncthreads();
    for (int v = threadIdx.x; v < 64 * kNRHS; v += blockDim.x) {
      const int jj = v / kNRHS, rr = v % kNRHS;
      sq[jj][swz_m<S>(jj, rr)] = j0 + jj < r ? Q[(br.slot + k + j0 + jj) * kNRHS + rr] : S{};
    }
    __syncthreads();
    const int jn = min(64, r - j0);
#pragma unroll 4
    for (int jj = 0; jj < jn; jj += 4) {
      const int jr = jj + kq;  // this lane's k index within the staged block
      double b[2][NP];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) parts3(sq[jr][swz_m<S>(jr, 8 * nb + rq)], b[nb]);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int i = rowi[mt], j = j0 + jr;
        double a[NP];
        parts3(i < k && j < r ? Tb[(int64_t)i * r + j] : S{}, a);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) dmma(C[mt][pp][nb][0], C[mt][pp][nb][1], a[pp], b[nb][pp]);
      }
    }
  }
  // lane holds rows rq (+8) and right-hand sides 2kq, 2kq+1 (+8)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int i = rowi[mt];
    if (i >= k || i >= it.first + kUpRowsM) continue;
    const int64_t dst = up_dst[br.skel + i];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int rhs = 8 * nb + 2 * kq + w;
        S v = Q[(br.slot + i) * kNRHS + rhs];
        if constexpr (CPLX) {
          const double t1 = C[mt][0][nb][w], t2 = C[mt][1][nb][w];
          v.x += t1 - t2;
          v.y += C[mt][2][nb][w] - t1 - t2;
        } else {
          v += C[mt][0][nb][w];
        }
        QH[(br.skel + i) * kNRHS + rhs] = v;
        Q[dst * kNRHS + rhs] = v;
      }
  }
}

static_assert(kDownColsM == 64, "K3m: four warps of 16 columns");

// K3m: uhat = UH + U[parent]; U_S += uhat (the item with first == 0);
// U_R[j][.] += sum_i conj(T[i,j]) uhat[i][.] for the item's 64 columns j.
template <class S>
__global__ void __launch_bounds__(128) k3m_downward(const LevelItem* __restrict__ items,
                                                    const BoxRec* __restrict__ box,
                                                    const int64_t* __restrict__ T_off,
                                                    const S* __restrict__ T, S* __restrict__ U,
                                                    const S* __restrict__ UH,
                                                    const int32_t* __restrict__ up_dst) {
  constexpr bool CPLX = sizeof(S) == 16;
  constexpr int NP = CPLX ? 3 : 1;
  extern __shared__ unsigned char smraw[];
  S* su = reinterpret_cast<S*>(smraw);  // [k rounded to 4][kNRHS], swizzled
  const LevelItem it = items[blockIdx.x];
  const BoxRec br = box[it.box];
  const int k = br.k, r = br.n - br.k;
  const int k4 = (k + 3) & ~3;
  for (int v = threadIdx.x; v < k4 * kNRHS; v += blockDim.x) {
    const int i = v / kNRHS, rr = v % kNRHS;
    S s{};
    if (i < k) {
      const S a = UH[(br.skel + i) * kNRHS + rr], b = U[(int64_t)up_dst[br.skel + i] * kNRHS + rr];
      if constexpr (CPLX) {
        s = make_double2(a.x + b.x, a.y + b.y);
      } else {
        s = a + b;
      }
      if (it.first == 0) {
        const S o = U[(br.slot + i) * kNRHS + rr];
        if constexpr (CPLX) {
          U[(br.slot + i) * kNRHS + rr] = make_double2(o.x + s.x, o.y + s.y);
        } else {
          U[(br.slot + i) * kNRHS + rr] = o + s;
        }
      }
    }
    su[i * kNRHS + swz_m<S>(i, rr)] = s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rq = lane >> 2, kq = lane & 3;
  const int jw = it.first + 16 * warp;  // this warp's 16 columns
  if (jw >= r) return;
  const S* Tb = T + T_off[it.box];
  double C[2][NP][2][2] = {};
#pragma unroll 4
  for (int i0 = 0; i0 < k; i0 += 4) {
    const int i = i0 + kq;
    double b[2][NP];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) parts3(su[i * kNRHS + swz_m<S>(i, 8 * nb + rq)], b[nb]);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int j = jw + 8 * mt + rq;
      S t = i < k && j < r ? Tb[(int64_t)i * r + j] : S{};
      if constexpr (CPLX) t.y = -t.y;  // conj(T)^T
      double a[NP];
      parts3(t, a);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) dmma(C[mt][pp][nb][0], C[mt][pp][nb][1], a[pp], b[nb][pp]);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int j = jw + 8 * mt + rq;
    if (j >= r) continue;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int rhs = 8 * nb + 2 * kq + w;
        S* o = U + (br.slot + k + j) * kNRHS + rhs;
        if constexpr (CPLX) {
          const double t1 = C[mt][0][nb][w], t2 = C[mt][1][nb][w];
          *o = make_double2(o->x + (t1 - t2), o->y + (C[mt][2][nb][w] - t1 - t2));
        } else {
          *o += C[mt][0][nb][w];
        }
      }
  }
}

// K2bm: the staged column sums of the symmetric u pass, added per receiving
// box in the plan's fixed (b, task, entry) order (deterministic); one CTA per
// box, consecutive threads on consecutive (point, rhs) scalars.
template <int SW>
__global__ void __launch_bounds__(256) k2bm_reduce(const BoxRec* __restrict__ box,
                                                   const int32_t* __restrict__ recv_box,
                                                   const int64_t* __restrict__ recv_off,
                                                   const int64_t* __restrict__ recv_u,
                                                   const double* __restrict__ St,
                                                   double* __restrict__ U) {
  constexpr int64_t kW = (int64_t)kNRHS * SW;  // scalars per point
  const BoxRec br = box[recv_box[blockIdx.x]];
  const int64_t e0 = recv_off[blockIdx.x], e1 = recv_off[blockIdx.x + 1];
  const int64_t len = (int64_t)br.n * kW;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int64_t e = e0; e < e1; ++e) s += __ldg(St + recv_u[e] * kW + i);
    U[br.slot * kW + i] += s;
  }
}

int grid_m(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// dynamic shared memory of the symmetric u pass: two generated blocks and the
// task's charges, 64 rows x 16 scalars each
constexpr size_t sym_smem_bytes(bool cplx) {
  return (size_t)3 * kMultiRows * kChunk * (cplx ? 2 : 1) * sizeof(double);
}

size_t k2m_smem(bool cplx, bool sym) { return sym ? sym_smem_bytes(cplx) : 0; }

template <int KER, bool TAB, bool TFO>
bool allow_sym_smem() {
  return cudaFuncSetAttribute(k2m_translate<KER, false, TAB, TFO, true>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sym_smem_bytes(KER == SFMM_HELMHOLTZ3D)) == cudaSuccess;
}

template <int KER, bool HPASS, bool SYM>
int blocks_per_sm() {
  constexpr bool CPLX = KER == SFMM_HELMHOLTZ3D;
  if (SYM && !(allow_sym_smem<KER, CPLX, false>() && allow_sym_smem<KER, CPLX, true>() &&
               allow_sym_smem<KER, false, false>() && allow_sym_smem<KER, false, true>()))
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, k2m_translate<KER, HPASS, CPLX, false, SYM>, kMThreads,
          k2m_smem(CPLX, SYM)) != cudaSuccess)
    return -1;
  return std::max(1, per_sm);
}

}  // namespace

int configure_multi(DevPlan& p, int device, size_t max_k, int max_entries) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  // the DMMA path holds a task's entry list in shared memory
  p.k2m_ok = max_entries <= kMEntCap ? 1 : 0;
  int bh, b0, bs;
  if (p.kernel == SFMM_HELMHOLTZ3D) {
    bh = blocks_per_sm<SFMM_HELMHOLTZ3D, true, false>();
    b0 = blocks_per_sm<SFMM_HELMHOLTZ3D, false, false>();
    bs = blocks_per_sm<SFMM_HELMHOLTZ3D, false, true>();
  } else if (p.kernel == SFMM_LAPLACE3D) {
    bh = blocks_per_sm<SFMM_LAPLACE3D, true, false>();
    b0 = blocks_per_sm<SFMM_LAPLACE3D, false, false>();
    bs = blocks_per_sm<SFMM_LAPLACE3D, false, true>();
  } else {
    bh = blocks_per_sm<SFMM_LAPLACE2D, true, false>();
    b0 = blocks_per_sm<SFMM_LAPLACE2D, false, false>();
    bs = blocks_per_sm<SFMM_LAPLACE2D, false, true>();
  }
  if (bh < 0 || b0 < 0 || bs < 0) return -1;
  p.k2m_grid = sms * bh;
  p.k2m_grid0 = sms * b0;
  p.k2m_grid_sym = sms * bs;
  const size_t sw = p.cplx ? 16 : 8;
  p.down_m_smem = std::max<size_t>(((max_k + 3) & ~(size_t)3) * kNRHS * sw, 16);
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
    k1m_upward<double2><<<(unsigned)(i1 - i0), 128, 0, st>>>(
        p.up_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.Q), reinterpret_cast<double2*>(s.QH), p.up_dst);
  else
    k1m_upward<double><<<(unsigned)(i1 - i0), 128, 0, st>>>(p.up_items + i0, p.box, p.T_off, p.T,
                                                             s.Q, s.QH, p.up_dst);
}

void launch_downward_m(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                       cudaStream_t st) {
  const int64_t i0 = hp.down_m_lvl[level], i1 = hp.down_m_lvl[level + 1];
  if (i1 <= i0) return;
  if (p.cplx)
    k3m_downward<double2><<<(unsigned)(i1 - i0), 128, p.down_m_smem, st>>>(
        p.down_m_items + i0, p.box, p.T_off, reinterpret_cast<const double2*>(p.T),
        reinterpret_cast<double2*>(s.U), reinterpret_cast<const double2*>(s.UH), p.up_dst);
  else
    k3m_downward<double><<<(unsigned)(i1 - i0), 128, p.down_m_smem, st>>>(
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
  a.X = p.X;
  a.Y = p.Y;
  a.Z = p.Z;
  a.sid = p.slot_id;
  a.Q = s.Q;
  a.QH = s.QH;
  a.U = s.U;
  a.UH = s.UH;
  a.err = p.err_flag;
  a.kappa = p.kappa;
  a.tab = p.sc_tab;
  a.ltab = p.log_tab;
  a.soff = p.ent_soff_m;
  a.stage = s.stage;
  a.sflag = s.stage_flags;
  const bool sym = p.multi_sym && s.stage != nullptr;
  cudaMemsetAsync(p.counter + 2, 0, 2 * sizeof(int), st);
  if (sym)
    cudaMemsetAsync(s.stage_flags, 0,
                    (size_t)(std::max<int64_t>(p.stage_m_points, kChunk) / kChunk) * sizeof(unsigned), st);
  // part 0: the u pass over every task (symmetric plans: the folded lists,
  // then K2bm); part 1: the uhat pass over the tasks that own skeleton rows
  // (unfolded lists, its own longest-first order)
  for (int part = 0; part < 2; ++part) {
    const int64_t t1 = part == 0 ? (sym ? p.n_tasks_msym : p.n_tasks_m) : p.n_tasks_mh;
    if (t1 <= 0) continue;
    const bool psym = sym && part == 0;
    a.tasks = part == 1 ? p.tasks_mh : (psym ? p.tasks_msym : p.tasks_m);
    a.er = psym ? p.ent_range_msym : p.ent_range_full;
    a.ent = psym ? p.entries_msym : p.entries_full;
    a.n_tasks = t1;
    a.counter = p.counter + 2 + part;
    const int grid =
        (int)std::min<int64_t>(part == 0 ? (psym ? p.k2m_grid_sym : p.k2m_grid0) : p.k2m_grid, t1);
    const size_t ssm = k2m_smem(p.cplx != 0, psym);
#define SFMM_K2M_LAUNCH(KER, TAB)                                                   \
  do {                                                                              \
    if (part == 1)                                                                  \
      k2m_translate<KER, true, TAB, false, false><<<grid, kMThreads, ssm, st>>>(a); \
    else if (psym && p.has_tfo_m)                                                   \
      k2m_translate<KER, false, TAB, true, true><<<grid, kMThreads, ssm, st>>>(a);  \
    else if (psym)                                                                  \
      k2m_translate<KER, false, TAB, false, true><<<grid, kMThreads, ssm, st>>>(a); \
    else if (p.has_tfo_m)                                                           \
      k2m_translate<KER, false, TAB, true, false><<<grid, kMThreads, ssm, st>>>(a); \
    else                                                                            \
      k2m_translate<KER, false, TAB, false, false><<<grid, kMThreads, ssm, st>>>(a);\
  } while (0)
    if (p.kernel == SFMM_HELMHOLTZ3D && p.sc_tab_ok)
      SFMM_K2M_LAUNCH(SFMM_HELMHOLTZ3D, true);
    else if (p.kernel == SFMM_HELMHOLTZ3D)
      SFMM_K2M_LAUNCH(SFMM_HELMHOLTZ3D, false);
    else if (p.kernel == SFMM_LAPLACE3D)
      SFMM_K2M_LAUNCH(SFMM_LAPLACE3D, false);
    else
      SFMM_K2M_LAUNCH(SFMM_LAPLACE2D, false);
#undef SFMM_K2M_LAUNCH
    if (psym && p.n_recv_m > 0) {
      if (p.cplx)
        k2bm_reduce<2><<<(unsigned)p.n_recv_m, 256, 0, st>>>(p.box, p.recv_m_box, p.recv_m_off,
                                                            p.recv_m_u, s.stage, s.U);
      else
        k2bm_reduce<1><<<(unsigned)p.n_recv_m, 256, 0, st>>>(p.box, p.recv_m_box, p.recv_m_off,
                                                            p.recv_m_u, s.stage, s.U);
    }
  }
}

}  // namespace sfmm_gpu
