// Kernel launchers of the sm_100a SRS-FMM apply (K0..K5).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan_build.h"

namespace sfmm_gpu {

// Per-apply device state for one right-hand side.  Scalars are double or
// interleaved complex (cplx = 1).
struct DevState {
  double* Q;    // slot charges        (n_slots scalars)
  double* QH;   // skeleton charges    (n_skel scalars)
  double* U;    // slot potentials     (n_slots scalars)
  double* UH;   // skeleton potentials (n_skel scalars)
  double* stage = nullptr;  // multi-RHS kSYM column sums (DevPlan::stage_m_points x kNRHS scalars)
  unsigned* stage_flags = nullptr;  // one chain flag per kChunkM staged points, zeroed per apply
};

struct DevPlan {
  int kernel, dim, cplx;
  double kappa;
  int64_t n_points, n_slots, n_skel;
  int32_t n_boxes, depth;
  BoxRec* box;
  EntryRange* ent_range;
  int32_t* entries;
  Task* tasks;
  int64_t n_tasks;
  int64_t n_interior;  // tasks[0, n_interior) read no ghost box
  double *X, *Y, *Z;
  int32_t* slot_id;
  int32_t* up_dst;     // skeleton entry -> slot of the same point in the parent
  int32_t* leaf_slot;  // owned point (slot order) -> slot
  int32_t* leaf_orig;  // owned point -> original index
  // single-rank plans with the two-pass K4 (k4_fold + k4_gather): original
  // index -> owned point (the inverse of leaf_orig), else null
  int32_t* leaf_pos = nullptr;
  // owned point of an uncompressed leaf (k = n, level >= 2) -> its skeleton
  // entry, else -1: K0 / K4 then also do that leaf's qhat copy / uhat fold
  // (the leaf-level k1_copy / k3_copy fused into the gather / scatter)
  int32_t* leaf_hat;
  double* T;
  int64_t* T_off;
  double2* sc_tab;  // (cos, sin)(k pi/128), 256 entries (fastmath.cuh)
  bool sc_tab_ok;   // kappa * (point-set diameter) within the table's reduction range
  double* log_tab;  // 3 x 128 doubles (fastmath.cuh fill_log_table)
  LevelItem *up_items, *down_items, *up1_items;  // up1: K1 (single rhs), up: K1m
  int32_t* copy_boxes;                            // warp-per-box lists (plan_build.h): upward
  int32_t* copy_boxes_dn;                         //   and downward
  double* orig_pts;
  double* stage;    // kSYM column-sum staging (stage_size scalars; one vector per pair)
  unsigned* stage_flags;  // stage_size / 32 chain flags (tiles that have added), zeroed per apply
  int sym_chain = 0;      // HostPlan::sym_chain: the chained K2 instantiation
  int32_t* recv_box;
  int64_t *recv_off, *recv_u, *recv_h;
  int64_t n_recv;
  int64_t* pack_idx;    // ghost exchange element indices into [Q | QH]
  int64_t* unpack_idx;
  int64_t n_pack, n_unpack;
  // cross-rank symmetric pairs (HostPlan::xsym): the second exchange
  int64_t *xpair_tile_off, *xtile_u, *xtile_h, *xpair_dst;
  int32_t *xpair_nu, *xpair_nh;
  int64_t n_xpairs;
  int64_t stage_size;      // local staging; received column sums follow it
  int64_t n_send2, n_recv2;
  int64_t n_owned_points;  // entries of leaf_slot / leaf_orig
  // multi-RHS path (kernels_multi.cu)
  EntryRange* ent_range_full;
  int32_t* entries_full;
  Task* tasks_m;
  int64_t n_tasks_m;
  LevelItem* down_m_items;
  Task* tasks_mh;      // the uhat pass's tasks (own skeleton rows)
  int64_t n_tasks_mh;
  int has_tfo_m = 0;   // entries_full holds tfo entries (K2m u pass needs qhat too)
  int k2m_grid, k2m_grid0;
  int k2m_ok = 1;        // every entry list fits K2m's shared memory (else the column loop)
  size_t down_m_smem;
  // symmetric multi-RHS u pass (HostPlan::multi_sym; staging in DevState::stage)
  int multi_sym = 0;
  EntryRange* ent_range_msym;
  int32_t *entries_msym, *ent_soff_m;
  Task* tasks_msym;
  int64_t n_tasks_msym = 0;
  int64_t stage_m_points = 0;
  int32_t* recv_m_box;
  int64_t *recv_m_off, *recv_m_u;
  int64_t n_recv_m = 0;
  int k2m_grid_sym = 0;
  int* counter;     // K2 task counters (interior, boundary, multi; reset per launch)
  int* err_flag;    // sticky duplicate-point flag
  int k2_grid;      // persistent K2 CTAs
  int k2_r1 = 0;    // every K2 task has <= 32 rows: the 64-register R = 1 kernel
  int k2_merged = 0;  // some K2 tasks are a box's merged row tiles (plan_build.cpp)
  size_t up_smem, down_smem;
  int k1_bulk = 0;          // real K1 stages T through cp.async.bulk (k1_upward_real_bulk)
  size_t up_bulk_smem = 0;
  int up_bulk_qr = 0;       // q_R doubles per ring stage
  int k1_bulk_grid = 148;   // persistent CTAs (one per SM)
  // persistent tree passes (HostPlan::tree_persist)
  int tree_persist = 0;
  TreeJob *up_jobs = nullptr, *down_jobs = nullptr;
  int32_t *up_stage_first = nullptr, *down_stage_first = nullptr;  // jobs before each stage
  int64_t n_up_jobs = 0, n_down_jobs = 0;
  int* tree_sync = nullptr;  // [up counter, down counter, up done, down done]
  int persist_grid = 0;
  size_t persist_smem = 0;
};

// K0: Q[leaf_slot[t]] = q[leaf_orig[t]] (+ the uncompressed leaves' qhat copy)
void launch_gather(const DevPlan& p, const double* q, DevState& s, cudaStream_t st);
// K1: one tree level of the upward pass (level >= 2)
void launch_upward(const DevPlan& p, const HostPlan& hp, int level, DevState& s, cudaStream_t st);
// K2: fused ifo/ifs/tfo/level-1 translation, all levels in one launch (or the
// interior / boundary halves of a sharded plan), followed by K2b
enum TranslatePart { kAllTasks, kInteriorTasks, kBoundaryTasks };
void launch_translate(const DevPlan& p, DevState& s, cudaStream_t st,
                      TranslatePart part = kAllTasks, bool reduce = true);
// K2b alone (after the second exchange of a cross-symmetric sharded plan)
void launch_stage_reduce(const DevPlan& p, DevState& s, cudaStream_t st);
// second exchange: buf[xpair_dst[i] + j] = sum over the pair's row tiles of
// the staged column sums (u part, then h part)
void launch_xpack(const DevPlan& p, double* buf, cudaStream_t st);
// ghost exchange: buf[i] = [Q | QH][pack_idx[i]]  /  [Q | QH][unpack_idx[i]] = buf[i]
void launch_pack(const DevPlan& p, const DevState& s, double* buf, cudaStream_t st);
void launch_unpack(const DevPlan& p, DevState& s, const double* buf, cudaStream_t st);
// K0 + K1 of every level (one launch per level, or one persistent launch for
// small plans) / K3 of every level + K4
void launch_upward_all(const DevPlan& p, const HostPlan& hp, const double* q, DevState& s,
                       cudaStream_t st);
void launch_downward_all(const DevPlan& p, const HostPlan& hp, DevState& s, double* u,
                         cudaStream_t st);
// K3: one tree level of the downward pass (level >= 2)
void launch_downward(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                     cudaStream_t st);
// K4: u[leaf_orig[t]] = U[leaf_slot[t]]
void launch_scatter(const DevPlan& p, const DevState& s, double* u, cudaStream_t st);
// K5: dense sum over all points in original order (depth < 2 fallback)
void launch_direct_fallback(const DevPlan& p, const double* q, double* u, cudaStream_t st);
// Dense subset sum for accuracy checks: one CTA per target.
void launch_direct_subset(int kernel, double kappa, int dim, int64_t n, const double* pts,
                          const double* q, int64_t nt, const int32_t* targets, double* u,
                          int* err_flag, cudaStream_t st);

// Device-side plan build: slot geometry/ids, upward destinations and the leaf
// maps from the uploaded index arrays (kernels_tree.cu).
struct SlotBuildArgs {
  const BoxRec* box;
  int64_t n_boxes;
  const int32_t* posmap;        // n_slots
  const int32_t* iv;            // n_slots, tree-order point ids
  const double* pts;            // tree order, interleaved
  int dim;
  const int32_t* parent;        // n_boxes
  const int32_t* parent_offset; // n_boxes
  const int32_t* leaf_box;      // owned leaves
  const int64_t* leaf_begin;
  const int64_t* leaf_out;
  int64_t n_leaves;
  const int32_t* perm;          // n_points
  double *X, *Y, *Z;
  int32_t* slot_id;
  int32_t* up_dst;
  int32_t* leaf_slot;
  int32_t* leaf_orig;
  int32_t* leaf_hat;
  const uint8_t* leaf_copy;     // owned leaf is uncompressed (its copies fused into K0/K4)
};
void launch_build_slots(const SlotBuildArgs& a, cudaStream_t st);
void launch_invert_orig(const DevPlan& p, int32_t* pos, cudaStream_t st);

// Persistent-grid size and dynamic shared memory setup (called at plan creation).
int configure_translate(DevPlan& p, int device);
int configure_tree_kernels(DevPlan& p, size_t max_r, size_t max_k);

// Multi-RHS passes over kNRHS right-hand sides at once (state stride kNRHS);
// nc <= kNRHS live columns, the rest are zero padding.
int configure_multi(DevPlan& p, int device, size_t max_k, int max_entries);
void launch_gather_m(const DevPlan& p, const double* q, int nc, DevState& s, cudaStream_t st);
void launch_upward_m(const DevPlan& p, const HostPlan& hp, int level, DevState& s, cudaStream_t st);
void launch_translate_m(const DevPlan& p, DevState& s, cudaStream_t st);
void launch_downward_m(const DevPlan& p, const HostPlan& hp, int level, DevState& s,
                       cudaStream_t st);
void launch_scatter_m(const DevPlan& p, const DevState& s, double* u, int nc, cudaStream_t st);


}  // namespace sfmm_gpu
