// Host-side flattening of an sfmm_plan_desc into the device layout.
//
// The reference keeps per-box std::vectors (ApplyPlan::x/xs/sid,
// ExpansionState::q/u/qhat/uhat; apply.hpp:22-42) and walks the neighbor
// lists phase by phase (apply.cpp:148-266).  The GPU plan instead owns a few
// flat arrays that stay resident in HBM:
//   * slot arrays (one entry per index_vec entry of every box), ordered
//     per box as [skeleton | redundant] so qhat/uhat are the first k slots;
//   * one translation CSR per target box covering all four phases;
//   * a cost-sorted task list for the persistent translation kernel;
//   * per-level work lists for the upward/downward interpolation GEMVs.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "sfmm_gpu.h"

namespace sfmm_gpu {

constexpr int kRowsPerLane = 4;                 // max rows per lane in K2
constexpr int kTileRows = 32 * kRowsPerLane;    // rows per K2 task
constexpr int kUpRows = 64;                     // K1m rows (skeleton entries) per CTA (4 warps x 16)
#ifndef SFMM_K1_ROWS
#define SFMM_K1_ROWS 64
#endif
constexpr int kUpRows1 = SFMM_K1_ROWS;          // K1 (single rhs) rows per CTA
constexpr int kDownCols = 256;                  // K3 columns (redundant slots) per CTA
constexpr int kChunkM = 16;                     // K2m sources per staged chunk
constexpr int kWarpBoxR = 32;                   // K1/K3: boxes with r <= this run warp per box
// a tree level's warp-per-box work and interpolation items in one launch
// (k_level): upward yes, downward no (measured, kernels_tree.cu)
#ifndef SFMM_K1_MERGE
#define SFMM_K1_MERGE 1
#endif
#ifndef SFMM_K3_MERGE
#define SFMM_K3_MERGE 0
#endif
constexpr int kMultiRows = 64;                  // K2m rows per task (4 warps x two 8-row DMMA tiles)
constexpr int kDownColsM = 64;                  // K3m columns per CTA (4 warps x 16)

struct LevelItem {
  int32_t box;
  int32_t first;  // first row (K1) / column (K3) of the chunk
};

// One job of the persistent tree passes (small plans, launch-bound): the
// whole upward pass -- K0 gather, then every level deepest first -- or the
// whole downward pass -- every level coarsest first, then K4 scatter -- in one
// launch; a job of stage s starts once every job of stage s - 1 has finished.
enum TreeJobKind : int32_t {
  kJobGather = 0,   // K0 on owned points [a * kPointsPerJob, +kPointsPerJob)
  kJobCopy = 1,     // k1_copy / k3_copy on copy_boxes[a, a + b)
  kJobItem = 2,     // K1 on up1_items[a] / K3 on down_items[a]
  kJobScatter = 3,  // K4 on owned points [a * kPointsPerJob, +kPointsPerJob)
};
constexpr int kPointsPerJob = 256;  // one point per thread
// plans with at most this many owned points run the persistent tree passes
// by default: none -- measured slower than the per-level launches replayed
// from a CUDA graph even on config 1 (profiles/r02/tree_persist_ab.txt), so
// they are an opt-in (SFMM_TREE_PERSIST=1)
constexpr int64_t kTreePersistPoints = 0;
struct TreeJob {
  int32_t kind, stage, a, b;
};

constexpr int32_t kShared = -1;  // HostPlan::owner of boxes every rank evaluates

struct HostPlan {
  int kernel = 0, dim = 0, cplx = 0;
  double kappa = 0;
  int64_t n_points = 0;
  int32_t n_boxes = 0, depth = 0;
  int64_t n_slots = 0, n_skel = 0, m_proj = 0;
  std::vector<int32_t> level_begin;
  std::vector<BoxRec> box;
  std::vector<int32_t> box_parent, box_level;
  std::vector<int64_t> T_off;                 // scalars
  // index_vec position -> slot offset inside its box ([skeleton | redundant],
  // a permutation per box).  The device derives the slot geometry (X, Y, Z,
  // slot_id), the upward destinations and the leaf gather/scatter maps from it
  // (launch_build_slots); the host never materialises them.
  std::vector<int32_t> posmap;
  std::vector<int32_t> parent_offset;         // box_parent_offset
  // owned leaves: box, first tree-order point, offset into leaf_slot/leaf_orig
  std::vector<int32_t> leaf_box;
  std::vector<int64_t> leaf_begin, leaf_out;  // leaf_out: leaf_box.size() + 1
  std::vector<uint8_t> leaf_copy;             // per owned leaf: uncompressed (k = n, level >= 2)
  // translation CSR and tasks
  std::vector<EntryRange> ent_range;
  std::vector<int32_t> entries;               // (src box << kModeBits) | mode
  std::vector<Task> tasks;
  int tile_rows = kTileRows;                  // K2 row-tile height chosen for this plan
  // symmetric colleague blocks: staged column sums and, per receiving box,
  // the staging slots to add (u part, and uhat part or -1) in a fixed order
  bool symmetric = false;
  bool sym_chain = false;                     // PlanOptions::sym_chain
  int64_t stage_size = 0;                     // scalars, a multiple of 32
  std::vector<int32_t> recv_box;
  std::vector<int64_t> recv_off;              // recv_box.size() + 1
  std::vector<int64_t> recv_u, recv_h;
  int64_t n_skipped_pairs = 0;                // cancelling pairs not evaluated
  int64_t n_split_parts = 0;                  // later parts of source-range split tasks
  int64_t n_merged_tasks = 0;                 // boxes whose row tiles run as one task (K2)
  int64_t n_interior_tasks = 0;               // tasks[0, n_interior) read no ghost box
  // sharding: owner rank of every box (whole subtrees at the cut
  // level; kShared: internal boxes above the cut, evaluated on every rank)
  int n_ranks = 1, rank = 0, cut_level = 1;
  std::vector<int32_t> owner;
  int64_t n_owned_points = 0;
  double p_dense_local = 0;                   // dense pairs this rank evaluates
  // ghost exchange: element indices into [Q | QH] (QH at offset n_slots),
  // per peer ranges send_off[p]..send_off[p+1] / recv_off_peer[p]..
  std::vector<int64_t> pack_idx, unpack_idx, send_off, recv_off_peer;
  // compact slot space (PlanOptions::compact, sharded plans): the descriptor's
  // slot / skeleton offset of every box (empty when not compacted), the runs
  // (global offset, compact offset, length) of index_vec entries to upload,
  // and the exchange lists in the descriptor's numbering (for describe)
  std::vector<int64_t> global_slot, global_skel;
  struct IvRun {
    int64_t src, dst, len;
  };
  std::vector<IvRun> iv_runs;
  std::vector<int64_t> pack_idx_global, unpack_idx_global;
  int64_t n_ghost_boxes = 0;
  // cross-rank symmetric pairs (PlanOptions::cross_symmetric).  Sender side:
  // group i (one receiving box c of one peer) sums the staged column sums of
  // its pairs over their row tiles xtile_u/xtile_h[xpair_tile_off[i] ..
  // xpair_tile_off[i+1]) (h: -1 = none) into the second send buffer at
  // xpair_dst[i] ([u: xpair_nu | h: xpair_nh] scalars), per destination rank
  // (send2_off).  Receiver side: the peer segments land at stage_size +
  // recv2_off[p] in the staging buffer and are listed in recv_u/recv_h after
  // the local column sums.
  bool xsym = false;
  std::vector<int64_t> xpair_tile_off, xtile_u, xtile_h, xpair_dst;
  std::vector<int32_t> xpair_nu, xpair_nh;
  std::vector<int64_t> send2_off, recv2_off;  // n_ranks + 1 each (scalars)
  // multi-RHS path: unfolded CSR (no kSYM), 16-row tasks, 16-column K3 items
  std::vector<EntryRange> ent_range_full;
  std::vector<int32_t> entries_full;
  std::vector<Task> tasks_m;                  // u pass, longest first
  std::vector<Task> tasks_mh;                 // uhat pass: the tasks owning skeleton rows,
  int64_t n_tasks_mh = 0;                     // longest first by their uhat-pass cost
  std::vector<LevelItem> down_m_items;
  std::vector<int64_t> down_m_lvl;
  // multi-RHS u pass with symmetric colleague blocks (single rank,
  // PlanOptions::multi_sym): the full CSR with each ifo pair of distinct
  // colleagues b < c folded into one kSYM entry of b; ent_soff_m[e] = first
  // point of entry e's staged vector within b's stage block (-1: not kSYM;
  // vectors are kChunkM-aligned).  Task::stage = b's stage block (points; each
  // staged point carries kNRHS scalars), Task::tile = the task's row tile
  // (tiles chain their column sums into one vector per pair).  K2bm adds, per
  // receiving box recv_m_box[i], the staged vectors recv_m_u[recv_m_off[i] ..
  // recv_m_off[i+1]) in that order.
  bool multi_sym = false;
  std::vector<EntryRange> ent_range_msym;
  std::vector<int32_t> entries_msym, ent_soff_m;
  std::vector<Task> tasks_msym;
  int64_t stage_m_points = 0;
  std::vector<int32_t> recv_m_box;
  std::vector<int64_t> recv_m_off, recv_m_u;
  // owned interpolation blocks copied from the descriptor into a compact blob
  struct Run {
    int64_t src, dst, len;  // scalars
  };
  std::vector<Run> T_runs;
  // interpolation work lists, concatenated per level; *_lvl has depth+2 entries
  std::vector<LevelItem> up_items, down_items, up1_items;
  std::vector<int64_t> up_lvl, down_lvl, up1_lvl;
  // owned boxes with k > 0 and no redundant slots (r = 0; the single-rhs
  // passes only copy qhat / fold uhat for them) or a short block
  // (r <= kWarpBoxR), per level: one warp per box (k1_copy, k3_copy)
  std::vector<int32_t> copy_boxes;
  std::vector<int64_t> copy_lvl;
  // the downward pass's warp-per-box list: uncompressed boxes only (a short
  // block's K3 keeps the column-per-thread CTA, measured faster there)
  std::vector<int32_t> copy_boxes_dn;
  std::vector<int64_t> copy_dn_lvl;
  // persistent tree passes (PlanOptions::tree_persist): job lists in stage
  // order and, per stage, the number of jobs in the stages before it
  bool tree_persist = false;
  std::vector<TreeJob> up_jobs, down_jobs;
  std::vector<int32_t> up_stage_first, down_stage_first;
  // depth < 2: coordinates in original order for the dense fallback
  std::vector<double> orig_pts;
  // stats
  int64_t n_ifo = 0, n_ifs = 0, n_tfo = 0, n_l1 = 0;
  double p_dense = 0, p_skel = 0;
};

// Validates the descriptor and fills `hp` for rank `rank` of `n_ranks`
// (1/0: the whole tree).  Returns SFMM_OK or an error code with a message in
// `err`.
// l1_owner (n_boxes, may be NULL): the rank of every level-1 box -- whole
// level-1 subtrees per rank, as chosen before the skeletons existed by a
// distributed precompute (subtree_owners) -- instead of the cost-based choice.
int build_host_plan(const sfmm_plan_desc& d, HostPlan& hp, std::string& err, int n_ranks = 1,
                    int rank = 0, int sym_chain = -1 /* -1: SFMM_SYM_CHAIN / SFMM_MERGE_TILES
                                                       (default per tile); 0 per tile;
                                                       1 chained; 2 merged tasks */,
                    const int32_t* l1_owner = nullptr);

// Tree-only ownership for a distributed precompute (no skeletons yet): the
// level-1 subtrees as Morton-contiguous ranges balancing the near-field work
// estimate sum over leaves of n_leaf * (points of its colleague leaves), so
// every rank can skeletonize exactly the subtrees it will own.  owner gets
// n_boxes entries (every box: its level-1 ancestor's rank; levels 0: -1).
int subtree_owners(int32_t n_boxes, const int32_t* level_begin, int32_t depth,
                   const int32_t* box_parent, const int32_t* box_begin, const int32_t* box_end,
                   const uint8_t* box_leaf, const int64_t* coll_off, const int32_t* coll,
                   int n_ranks, int32_t* owner, std::string& err);

// Plan options (environment SFMM_SYMMETRIC=0 / SFMM_SKIP_CANCEL=0 turn them off
// for A/B measurements; both default on).
struct PlanOptions {
  bool symmetric = true;    // evaluate each off-diagonal colleague block once
  bool skip_cancel = true;  // drop pairs whose add and subtract cancel exactly
  // sharded plans: true = run the interior tasks while the ghost exchange is in
  // flight (two translation launches); false (default) = exchange right after
  // the upward pass, then one launch over all tasks.  Measured (per-rank device
  // time, N=1e7): one launch 13.4 ms vs 15.9 ms at 8 ranks -- the second
  // launch's tail costs far more than the exposed exchange (~0.1 ms).
  bool overlap = false;
  // sharded symmetric plans: a colleague pair split across two ranks is
  // evaluated once, by one of the two owners (chosen to balance the ranks'
  // work), which returns the other side's column sums in a second (smaller)
  // exchange (SFMM_SHARD_XSYM=0: both ranks evaluate it, one exchange).
  bool cross_symmetric = true;
  // kSYM column sums of a box's row tiles chained into one staged vector per
  // pair (tile t adds to tile t-1's, in order) instead of one vector per
  // (pair, row tile): ~2/3 less staging memory at 1e7, but the tiles wait for
  // each other (K2 +19 % at 1e7), so it is used only when the plan would not
  // fit otherwise (sfmm_gpu.cu) or on request (SFMM_SYM_CHAIN=1).
  int sym_chain = 0;
  // per-tile layout: a box's row tiles as one merged task (its tiles in
  // order, one staged column-sum vector per pair: the chained layout's
  // memory without its waits) when the box costs at most merge_share of the
  // per-warp share of K2.  The low-memory layout tried first when the plan
  // would not fit (sfmm_gpu.cu); measured 3.8 % slower K2 than per-tile
  // staging at 1e7 (coarser tasks), so not the default (SFMM_MERGE_TILES=1).
  bool merge_tiles = false;
  double merge_share = 0.5;
  // multi-RHS apply: colleague blocks generated once for both directions
  // (the transposed DMMA product of K2m, column sums chained over b's row
  // tiles).  Opt-in (SFMM_MULTI_SYM=1): measured slower on config 4 (DESIGN.md
  // 3, profiles/r02/k2m_sym_ab.txt) -- K2m is DMMA-bound, the fold saves only
  // generation and costs occupancy and the tile chain's waits.
  bool multi_sym = false;
  // tree passes as two persistent launches (gather + upward levels, downward
  // levels + scatter) instead of one to three launches per level: -1 = for
  // plans of at most kTreePersistPoints points (SFMM_TREE_PERSIST=0/1 forces)
  int tree_persist = -1;
  // small single-rank real plans: cut the row tiles that would set K2's
  // makespan along their entry lists (SFMM_SPLIT=0 turns it off)
  bool split = true;
  double split_part = 0.5;  // part size as a fraction of the per-warp share (split above 1.5x it)
  // sharded plans: slots only for the boxes the rank touches (SFMM_SHARD_COMPACT=0: all N)
  bool compact = true;
};
PlanOptions plan_options_from_env();

}  // namespace sfmm_gpu
