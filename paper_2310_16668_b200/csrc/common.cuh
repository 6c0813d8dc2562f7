// Shared device-side types of the sm_100a SRS-FMM apply.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sfmm_gpu {

// Translation modes of one (target box, source box) entry of the fused
// translation CSR.  They are the four reference phases (apply.cpp:148-266).
enum Mode : int32_t {
  kIFO = 0,  // colleagues, level >= 2: u_b += A(B_b,B_c) q_c ; uhat_b -= A(S_b,S_c) qhat_c
  kIFS = 1,  // coarse leaves:          u_b += A(B_b,L_c) q_c ; uhat_b -= A(S_b,L_c) q_c
  kTFO = 2,  // fine boxes of a leaf:   u_b += A(L_b,B_c) q_c - A(L_b,S_c) qhat_c
  kL1 = 3,   // level-1 all pairs:      u_b += A(B_b,B_c) q_c
  kSYM = 4   // IFO with a colleague c > b, evaluated once for both directions:
             // b's rows as kIFO, c's rows (A_cb = A_bc^T) as staged column sums
};
constexpr int kNRHS = 16;  // right-hand sides per multi-RHS pass (zero padded)
// Largest rows-per-lane of the complex K2 (row tiles of complex plans are at
// most 32 x this; plan_build.cpp and kernels_translate.cu must agree).
#ifndef SFMM_K2C_MAX_R
#define SFMM_K2C_MAX_R 3
#endif
// Largest rows-per-lane of the real K2 (a build knob, tools/build_variant.sh):
// real row tiles are at most 32 x this (plan_build.cpp clamps them).
#ifndef SFMM_K2_MAX_R
#define SFMM_K2_MAX_R 4
#endif
static_assert(SFMM_K2_MAX_R >= 1 && SFMM_K2_MAX_R <= 4, "SFMM_K2_MAX_R must be 1..4");
static_assert(SFMM_K2C_MAX_R >= 2 && SFMM_K2C_MAX_R <= 4, "SFMM_K2C_MAX_R must be 2..4");
constexpr int kModeBits = 3;
constexpr int32_t kModeMask = (1 << kModeBits) - 1;

// Per-box record used by the translation kernel.  Slots of a compressed box
// are ordered [skeleton (skel_pos order) | redundant (red_pos order)], so
// qhat/uhat of box b line up with its first k slots.
struct BoxRec {
  int64_t slot;   // first slot of the box in the slot arrays
  int64_t skel;   // first entry of the box in the skeleton arrays (qhat/uhat)
  int32_t n;      // |index_vec|
  int32_t k;      // |skel_pos|
};

// One translation work item: rows [row0, row0+nrows) of target box `box`
// against every CSR entry of that box.  Each row has exactly one owner, so the
// kernel writes results with plain stores (no atomics, deterministic).
struct Task {
  int32_t box;
  int32_t row0;
  int32_t nrows;
  int32_t tile;   // row-tile index within the box (chained kSYM column sums), -1: unchained
  int64_t stage;  // first staging slot of the box's kSYM column sums
  // Source-range split of a long task (small plans, plan_build.cpp): entries
  // [e0, e1) of the box's list (e1 < 0: all), and the staging slot where a
  // part other than the first leaves its raw row partials (-1: the task owns
  // the rows and writes U / UH itself)
  int32_t e0 = 0;
  int32_t e1 = -1;
  int64_t rstage = -1;
};

struct EntryRange {
  int64_t begin;
  int32_t count;
  int32_t pad;
};

}  // namespace sfmm_gpu
