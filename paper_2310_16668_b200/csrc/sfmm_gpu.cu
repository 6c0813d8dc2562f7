// C ABI of the sm_100a SRS-FMM apply (include/sfmm_gpu.h).
//
// Orchestrates one apply exactly in the reference's phase order
// (fmm_apply, /root/reference/proj/src/apply.cpp:306-337):
//   K0 gather -> K1 upward (levels depth..2) -> K2 fused translation (one
//   launch: ifo, ifs, tfo, level-1) -> K3 downward (levels 2..depth) ->
//   K4 scatter;   depth < 2 -> K5 dense fallback.
// The plan (geometry, index maps, interpolation operators, translation CSR,
// task list) is uploaded once by sfmm_gpu_plan_create and stays resident.
#include "fastmath.cuh"
#include "plan.h"

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace sfmm_gpu {
int set_last_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace sfmm_gpu


extern "C" {

const char* sfmm_gpu_last_error(void) { return g_last_error.c_str(); }

const char* sfmm_gpu_version(void) { return "sfmm_gpu 0.1 (sm_100a, FP64)"; }

}  // extern "C"

namespace sfmm_gpu {

// T_dev: the descriptor's operators in device memory (global T_off layout), or
// with T_compact only the owned runs concatenated (sfmm_gpu_shard_T_runs order)
int create_plan(const sfmm_plan_desc* desc, int device, int n_ranks, int rank,
                sfmm_gpu_plan** out, const double* T_dev, bool T_compact,
                std::shared_ptr<double> T_share, const int32_t* l1_owner) {
  if (!desc || !out) return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create: null argument");
  *out = nullptr;
  sfmm_gpu_plan* p = nullptr;
  try {
    p = new sfmm_gpu_plan();
    std::string err;
    int rc = build_host_plan(*desc, p->hp, err, n_ranks, rank, -1, l1_owner);
    if (rc != SFMM_OK) {
      delete p;
      return set_error(rc, err);
    }
    p->device = device;
    DeviceGuard device_guard(device);
    // Per-tile kSYM staging is the fast layout; when the plan would not fit
    // the free device memory with it, merge each box's row tiles into one task
    // with one staged vector per pair (PlanOptions::merge_tiles), and if that
    // still does not fit, chain the row tiles' column sums (sym_chain)
    if (!p->hp.sym_chain && p->hp.n_merged_tasks == 0 && p->hp.stage_size > 0 &&
        !std::getenv("SFMM_SYM_CHAIN") && !std::getenv("SFMM_MERGE_TILES")) {
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        auto need_of = [&](const HostPlan& h) {
          const double sw = h.cplx ? 2.0 : 1.0;
          double need = 8.0 * sw * ((double)h.stage_size + 2.0 * h.n_slots + 2.0 * h.n_skel) +
                        28.0 * h.n_slots + 16.0 * h.n_owned_points + 8.0 * h.n_skel +
                        24.0 * (double)h.tasks.size() + 4.0 * (double)h.entries.size();
          if (!(T_dev && !T_compact && n_ranks == 1)) need += 8.0 * sw * (double)h.T_off.back();
          return need;
        };
        const double avail = 0.92 * (double)free_b;
        for (int layout : {2, 1}) {  // merged tasks, then chained
          if (need_of(p->hp) <= avail) break;
          HostPlan lighter;
          if (build_host_plan(*desc, lighter, err, n_ranks, rank, layout, l1_owner) == SFMM_OK)
            p->hp = std::move(lighter);
        }
      }
    }
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreate(&p->ev_a), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_b), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_k2a), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_k2b), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(p->ev_done, p->stream), "event");
    HostPlan& hp = p->hp;
    DevPlan& dp = p->dp;
    dp.kernel = hp.kernel;
    dp.dim = hp.dim;
    dp.cplx = hp.cplx;
    dp.kappa = hp.kappa;
    dp.n_points = hp.n_points;
    dp.n_boxes = hp.n_boxes;
    dp.depth = hp.depth;
    dp.n_owned_points = hp.n_owned_points;
    dp.counter = p->alloc<int>(4);
    dp.err_flag = p->alloc<int>(4);
    ck(cudaMemset(dp.err_flag, 0, 4 * sizeof(int)), "memset");
    const int sw = hp.cplx ? 2 : 1;
    if (hp.depth < 2) {
      dp.orig_pts = p->upload(hp.orig_pts);
    } else {
      dp.n_slots = hp.n_slots;
      dp.n_skel = hp.n_skel;
      dp.box = p->upload(hp.box);
      dp.ent_range = p->upload(hp.ent_range);
      dp.entries = p->upload(hp.entries);
      dp.tasks = p->upload(hp.tasks);
      dp.n_tasks = (int64_t)hp.tasks.size();
      dp.n_interior = hp.n_interior_tasks;
      // slot geometry, upward destinations and leaf maps are built on the
      // device from the index arrays
      dp.X = p->alloc<double>(hp.n_slots);
      dp.Y = p->alloc<double>(hp.n_slots);
      dp.Z = p->alloc<double>(hp.n_slots);
      dp.slot_id = p->alloc<int32_t>(hp.n_slots);
      // slot indices are int32 on the device (12 B of maps per point in K0/K4)
      if (hp.n_slots >= (int64_t)INT32_MAX)
        throw CudaFail{SFMM_EUNSUPPORTED, "more than 2^31 slots in one plan: shard it"};
      dp.up_dst = p->alloc<int32_t>(hp.n_skel);
      dp.leaf_slot = p->alloc<int32_t>(hp.n_owned_points);
      dp.leaf_orig = p->alloc<int32_t>(hp.n_owned_points);
      dp.leaf_hat = p->alloc<int32_t>(hp.n_owned_points);
      {
        TmpDev tmp;
        SlotBuildArgs a{};
        a.box = dp.box;
        a.n_boxes = hp.n_boxes;
        a.posmap = tmp.up(hp.posmap.data(), hp.posmap.size());
        if (hp.iv_runs.empty()) {
          a.iv = tmp.up(desc->iv, (size_t)hp.n_slots);
        } else {  // compact slot space: the present boxes' index_vec runs
          std::vector<int32_t> iv((size_t)hp.n_slots);
          for (const HostPlan::IvRun& r : hp.iv_runs)
            std::copy(desc->iv + r.src, desc->iv + r.src + r.len, iv.begin() + r.dst);
          a.iv = tmp.up(iv.data(), iv.size());
        }
        a.pts = tmp.up(desc->pts, (size_t)hp.n_points * hp.dim);
        a.dim = hp.dim;
        a.parent = tmp.up(hp.box_parent.data(), hp.box_parent.size());
        a.parent_offset = tmp.up(hp.parent_offset.data(), hp.parent_offset.size());
        a.leaf_box = tmp.up(hp.leaf_box.data(), hp.leaf_box.size());
        a.leaf_begin = tmp.up(hp.leaf_begin.data(), hp.leaf_begin.size());
        a.leaf_out = tmp.up(hp.leaf_out.data(), hp.leaf_out.size());
        a.leaf_copy = tmp.up(hp.leaf_copy.data(), hp.leaf_copy.size());
        a.n_leaves = (int64_t)hp.leaf_box.size();
        a.perm = tmp.up(desc->perm, (size_t)hp.n_points);
        a.X = dp.X;
        a.Y = dp.Y;
        a.Z = dp.Z;
        a.slot_id = dp.slot_id;
        a.up_dst = dp.up_dst;
        a.leaf_slot = dp.leaf_slot;
        a.leaf_orig = dp.leaf_orig;
        a.leaf_hat = dp.leaf_hat;
        launch_build_slots(a, p->stream);
        ck(cudaGetLastError(), "build slots");
        // single-rank plans whose potentials outgrow L2's reach: K4 as fold +
        // original-order gather (kernels_tree.cu k4_fold / k4_gather).  A/B
        // (profiles/r02/k4_gather_ab.txt): 0.252 -> 0.148 ms at 1e7, but
        // 0.016 -> 0.026 ms at 1e6, where the scatter's lines stay in L2.
        // SFMM_K4_GATHER=1 / 0 forces it on / off.
        const char* kg = std::getenv("SFMM_K4_GATHER");
        const bool big = (double)hp.n_points * 8.0 * sw >= 24e6;
        if (hp.n_owned_points == hp.n_points && hp.n_points > 0 &&
            (kg ? kg[0] == '1' : big)) {
          dp.leaf_pos = p->alloc<int32_t>(hp.n_owned_points);
          launch_invert_orig(dp, dp.leaf_pos, p->stream);
          ck(cudaGetLastError(), "invert leaf map");
        }
        ck(cudaStreamSynchronize(p->stream), "build slots");
      }
      dp.T_off = p->upload(hp.T_off);
      {
        std::vector<double2> tab(kSinCosTab);
        fill_sincos_table(tab.data());
        dp.sc_tab = p->upload(tab);
        // every kernel argument kappa * r is at most kappa * (bounding-box diagonal)
        double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int k = 0; k < hp.dim; ++k) lo[k] = hi[k] = desc->pts[k];
        for (int64_t i = 0; i < hp.n_points; ++i)
          for (int k = 0; k < hp.dim; ++k) {
            lo[k] = std::min(lo[k], desc->pts[i * hp.dim + k]);
            hi[k] = std::max(hi[k], desc->pts[i * hp.dim + k]);
          }
        double d2 = 0;
        for (int k = 0; k < hp.dim; ++k) d2 += (hi[k] - lo[k]) * (hi[k] - lo[k]);
        dp.sc_tab_ok = std::fabs(hp.kappa) * std::sqrt(d2) <= kSinCosTabMaxArg;
        std::vector<double> lt(kLogTabLen);
        fill_log_table(lt.data());
        dp.log_tab = p->upload(lt);
      }
      // interpolation operators of the owned boxes, copied run by run
      // A single-rank plan built from device operators in the descriptor's
      // layout keeps that buffer (shared with the skeletonization result)
      // instead of copying it: at N = 1e8 the copy alone would need ~96 GB more.
      bool identity = T_share && T_dev && !T_compact && n_ranks == 1 &&
                      T_share.get() == T_dev;
      for (const HostPlan::Run& r : hp.T_runs) identity = identity && r.src == r.dst;
      if (identity) {
        p->T_hold = T_share;
        dp.T = T_share.get();
        p->device_bytes += (int64_t)(sizeof(double) * hp.T_off[hp.n_boxes] * sw);
      } else {
        // (+2: K1's bulk copies round each row range out to 16-byte boundaries)
        dp.T = p->alloc<double>((size_t)hp.T_off[hp.n_boxes] * sw + 2);
      }
      // device operators may still be in flight on another stream (a pack on
      // the legacy stream, an NCCL receive): the plan's stream is non-blocking.
      // They may live on another device (sfmm_gpu_plan_create_multi_skel):
      // the copies below are then peer copies (cudaMemcpyDefault, UVA).
      if (T_dev) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, T_dev) == cudaSuccess && attr.device >= 0 &&
            attr.device != device) {
          DeviceGuard g2(attr.device);
          ck(cudaDeviceSynchronize(), "wait for T");
        }
        ck(cudaDeviceSynchronize(), "wait for T");
      }
      const double* T_src = T_dev ? T_dev : desc->T;
      if (!T_src && !hp.T_runs.empty()) throw CudaFail{SFMM_EINVAL, "descriptor has no T"};
      for (const HostPlan::Run& r : hp.T_runs) {
        if (identity) break;
        ck(cudaMemcpyAsync(dp.T + r.dst * sw, T_src + (T_compact ? r.dst : r.src) * sw,
                           sizeof(double) * r.len * sw,
                           T_dev ? cudaMemcpyDefault : cudaMemcpyHostToDevice, p->stream),
           "upload T");
      }
      ck(cudaStreamSynchronize(p->stream), "upload T");
      dp.up_items = p->upload(hp.up_items);
      dp.up1_items = p->upload(hp.up1_items);
      dp.copy_boxes = p->upload(hp.copy_boxes);
      dp.copy_boxes_dn = p->upload(hp.copy_boxes_dn);
      dp.down_items = p->upload(hp.down_items);
      if (hp.tree_persist) {
        dp.tree_persist = 1;
        dp.up_jobs = p->upload(hp.up_jobs);
        dp.down_jobs = p->upload(hp.down_jobs);
        dp.n_up_jobs = (int64_t)hp.up_jobs.size();
        dp.n_down_jobs = (int64_t)hp.down_jobs.size();
        dp.up_stage_first = p->upload(hp.up_stage_first);
        dp.down_stage_first = p->upload(hp.down_stage_first);
        dp.tree_sync = p->alloc<int>(4);
      }
      const int64_t n_recv2 = hp.recv2_off.empty() ? 0 : hp.recv2_off.back();
      dp.stage_size = hp.stage_size;
      dp.sym_chain = hp.sym_chain ? 1 : 0;
      dp.n_recv2 = n_recv2;
      dp.n_send2 = hp.send2_off.empty() ? 0 : hp.send2_off.back();
      dp.stage = p->alloc<double>((size_t)std::max<int64_t>(hp.stage_size + n_recv2, 1) * sw);
      // row partials of split tasks: rows outside a part's tile are never
      // written and must read as zero in K2b
      if (hp.n_split_parts > 0)
        ck(cudaMemset(dp.stage, 0, sizeof(double) * (size_t)(hp.stage_size + n_recv2) * sw),
           "zero staging");
      dp.stage_flags = p->alloc<unsigned>((size_t)std::max<int64_t>(hp.stage_size >> 5, 1));
      dp.n_xpairs = (int64_t)hp.xpair_dst.size();
      dp.xpair_tile_off = p->upload(hp.xpair_tile_off);
      dp.xtile_u = p->upload(hp.xtile_u);
      dp.xtile_h = p->upload(hp.xtile_h);
      dp.xpair_dst = p->upload(hp.xpair_dst);
      dp.xpair_nu = p->upload(hp.xpair_nu);
      dp.xpair_nh = p->upload(hp.xpair_nh);
      dp.n_recv = (int64_t)hp.recv_box.size();
      dp.recv_box = p->upload(hp.recv_box);
      dp.recv_off = p->upload(hp.recv_off);
      dp.recv_u = p->upload(hp.recv_u);
      dp.recv_h = p->upload(hp.recv_h);
      dp.ent_range_full = p->upload(hp.ent_range_full);
      dp.entries_full = p->upload(hp.entries_full);
      dp.tasks_m = p->upload(hp.tasks_m);
      for (int32_t c : hp.entries_full) dp.has_tfo_m |= (c & kModeMask) == kTFO ? 1 : 0;
      dp.n_tasks_m = (int64_t)hp.tasks_m.size();
      dp.n_tasks_mh = hp.n_tasks_mh;
      dp.tasks_mh = p->upload(hp.tasks_mh);
      dp.down_m_items = p->upload(hp.down_m_items);
      if (hp.multi_sym) {
        dp.multi_sym = 1;
        dp.ent_range_msym = p->upload(hp.ent_range_msym);
        dp.entries_msym = p->upload(hp.entries_msym);
        dp.ent_soff_m = p->upload(hp.ent_soff_m);
        dp.tasks_msym = p->upload(hp.tasks_msym);
        dp.n_tasks_msym = (int64_t)hp.tasks_msym.size();
        dp.stage_m_points = hp.stage_m_points;
        dp.recv_m_box = p->upload(hp.recv_m_box);
        dp.recv_m_off = p->upload(hp.recv_m_off);
        dp.recv_m_u = p->upload(hp.recv_m_u);
        dp.n_recv_m = (int64_t)hp.recv_m_box.size();
      }
      dp.pack_idx = p->upload(hp.pack_idx);
      dp.unpack_idx = p->upload(hp.unpack_idx);
      dp.n_pack = (int64_t)hp.pack_idx.size();
      dp.n_unpack = (int64_t)hp.unpack_idx.size();
      size_t max_r = 0, max_k = 0;
      for (const BoxRec& b : hp.box) {
        max_r = std::max<size_t>(max_r, (size_t)(b.n - b.k));
        max_k = std::max<size_t>(max_k, (size_t)b.k);
      }
      if (configure_tree_kernels(dp, max_r, max_k) != 0)
        throw CudaFail{SFMM_EUNSUPPORTED, "interpolation block too large for shared memory"};
      {
        int32_t max_rows = 0;
        for (const Task& t : hp.tasks) max_rows = std::max(max_rows, t.nrows);
        dp.k2_r1 = !hp.cplx && max_rows <= 32;
        dp.k2_merged = hp.n_merged_tasks > 0 ? 1 : 0;
        if (dp.k2_merged && (dp.k2_r1 || hp.sym_chain))
          throw CudaFail{SFMM_EINVAL, "merged K2 tasks with a 32-row or chained plan"};
      }
      if (configure_translate(dp, device) != 0)
        throw CudaFail{SFMM_ECUDA, "occupancy query failed"};
      int max_entries = 0;
      for (const EntryRange& e : hp.ent_range_full) max_entries = std::max(max_entries, e.count);
      for (const EntryRange& e : hp.ent_range_msym) max_entries = std::max(max_entries, e.count);
      if (configure_multi(dp, device, max_k, max_entries) != 0)
        throw CudaFail{SFMM_EUNSUPPORTED, "multi-RHS configuration failed"};
      p->ds.Q = p->alloc<double>((size_t)hp.n_slots * sw);
      p->ds.U = p->alloc<double>((size_t)hp.n_slots * sw);
      p->ds.QH = p->alloc<double>((size_t)hp.n_skel * sw);
      p->ds.UH = p->alloc<double>((size_t)hp.n_skel * sw);
      // release host copies that now live on the device
      std::vector<int32_t>().swap(hp.posmap);
      std::vector<int32_t>().swap(hp.entries);
      std::vector<Task>().swap(hp.tasks);
      std::vector<int32_t>().swap(hp.entries_full);
      std::vector<Task>().swap(hp.tasks_m);
      std::vector<Task>().swap(hp.tasks_mh);
      std::vector<EntryRange>().swap(hp.ent_range_msym);
      std::vector<int32_t>().swap(hp.entries_msym);
      std::vector<int32_t>().swap(hp.ent_soff_m);
      std::vector<Task>().swap(hp.tasks_msym);
      std::vector<int64_t>().swap(hp.recv_m_u);
      std::vector<int64_t>().swap(hp.pack_idx);
      std::vector<int64_t>().swap(hp.unpack_idx);
    }
    ck(cudaDeviceSynchronize(), "plan upload");
    *out = p;
    return SFMM_OK;
  } catch (const CudaFail& f) {
    delete p;
    return set_error(f.code, "sfmm_gpu_plan_create: " + f.msg);
  } catch (const std::bad_alloc&) {
    delete p;
    return set_error(SFMM_ENOMEM, "sfmm_gpu_plan_create: host allocation failed");
  }
}

}  // namespace sfmm_gpu

namespace sfmm_gpu {
namespace {

// apply_end = mid + fin; the second exchange in between exists only for
// cross-symmetric sharded plans
void apply_mid_impl(sfmm_gpu_plan* p, const void* recv_dev, void* send2_dev, cudaStream_t st) {
  if (p->hp.depth < 2) return;
  if (p->dp.n_unpack > 0) {
    if (!recv_dev) throw CudaFail{SFMM_EINVAL, "receive buffer required"};
    launch_unpack(p->dp, p->ds, static_cast<const double*>(recv_dev), st);
  }
  launch_translate(p->dp, p->ds, st, kBoundaryTasks, false);
  if (p->dp.n_xpairs > 0) {
    if (!send2_dev) throw CudaFail{SFMM_EINVAL, "second send buffer required"};
    launch_xpack(p->dp, static_cast<double*>(send2_dev), st);
  }
}

void apply_fin_impl(sfmm_gpu_plan* p, const void* q_dev, const void* recv2_dev, void* u_dev,
                    cudaStream_t st) {
  double* u = static_cast<double*>(u_dev);
  if (p->hp.depth < 2) {
    if (p->hp.rank == 0) launch_direct_fallback(p->dp, static_cast<const double*>(q_dev), u, st);
    return;
  }
  if (p->dp.n_recv2 > 0) {
    if (!recv2_dev) throw CudaFail{SFMM_EINVAL, "second receive buffer required"};
    const size_t sw = p->dp.cplx ? 2 : 1;
    ck(cudaMemcpyAsync(p->dp.stage + p->dp.stage_size * sw, recv2_dev,
                       sizeof(double) * p->dp.n_recv2 * sw, cudaMemcpyDeviceToDevice, st),
       "second exchange");
  }
  launch_stage_reduce(p->dp, p->ds, st);
  launch_downward_all(p->dp, p->hp, p->ds, u, st);
}

}  // namespace

// Phases of one sharded apply, shared by the C ABI's
// begin/mid/fin/end entry points and the in-library exchanges (sfmm_multi.cu).
// user_stream != NULL replays each phase as a CUDA graph keyed on its buffers.
void phase_begin(sfmm_gpu_plan* p, const void* q_dev, void* send_dev, void* user_stream,
                 cudaStream_t st, cudaEvent_t packed) {
  const double* q = static_cast<const double*>(q_dev);
  if (p->hp.depth >= 2 && p->dp.n_pack > 0 && !send_dev)
    throw CudaFail{SFMM_EINVAL, "send buffer required"};
  p->run_phase(0, q_dev, send_dev, nullptr, user_stream, st, [&] {
    if (p->hp.depth < 2) return;
    launch_upward_all(p->dp, p->hp, q, p->ds, st);
    if (p->dp.n_pack > 0) launch_pack(p->dp, p->ds, static_cast<double*>(send_dev), st);
  });
  if (packed) ck(cudaEventRecord(packed, st), "event");
  // zeroes U / UH (and, with SFMM_SHARD_OVERLAP=1, runs the interior tasks)
  if (p->hp.depth >= 2) launch_translate(p->dp, p->ds, st, kInteriorTasks);
}

void phase_mid(sfmm_gpu_plan* p, const void* recv_dev, void* send2_dev, void* user_stream,
               cudaStream_t st, cudaEvent_t packed) {
  if (p->hp.depth >= 2 && p->dp.n_unpack > 0 && !recv_dev)
    throw CudaFail{SFMM_EINVAL, "receive buffer required"};
  if (p->hp.depth >= 2 && p->dp.n_xpairs > 0 && !send2_dev)
    throw CudaFail{SFMM_EINVAL, "second send buffer required"};
  p->run_phase(1, recv_dev, send2_dev, nullptr, user_stream, st,
               [&] { apply_mid_impl(p, recv_dev, send2_dev, st); });
  if (packed) ck(cudaEventRecord(packed, st), "event");
}

void phase_fin(sfmm_gpu_plan* p, const void* q_dev, const void* recv2_dev, void* u_dev,
               void* user_stream, cudaStream_t st) {
  if (p->hp.depth >= 2 && p->dp.n_recv2 > 0 && !recv2_dev)
    throw CudaFail{SFMM_EINVAL, "second receive buffer required"};
  p->run_phase(2, q_dev, recv2_dev, u_dev, user_stream, st,
               [&] { apply_fin_impl(p, q_dev, recv2_dev, u_dev, st); });
}

void phase_end(sfmm_gpu_plan* p, const void* q_dev, const void* recv_dev, void* u_dev,
               void* user_stream, cudaStream_t st) {
  if (p->hp.depth >= 2 && p->dp.n_unpack > 0 && !recv_dev)
    throw CudaFail{SFMM_EINVAL, "receive buffer required"};
  p->run_phase(1, recv_dev, q_dev, u_dev, user_stream, st, [&] {
    apply_mid_impl(p, recv_dev, nullptr, st);
    apply_fin_impl(p, q_dev, nullptr, u_dev, st);
  });
}

}  // namespace sfmm_gpu

extern "C" {

int sfmm_gpu_plan_create(const sfmm_plan_desc* desc, int device, sfmm_gpu_plan** out) {
  return create_plan(desc, device, 1, 0, out);
}

int sfmm_gpu_plan_create_sharded(const sfmm_plan_desc* desc, int device, int n_ranks, int rank,
                                 sfmm_gpu_plan** out) {
  return create_plan(desc, device, n_ranks, rank, out);
}

int sfmm_gpu_plan_create_skel(const sfmm_plan_desc* desc, const sfmm_skel_result* skel,
                              int device, int n_ranks, int rank, sfmm_gpu_plan** out) {
  if (!desc || !skel || !out) return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_skel: null argument");
  int skel_dev = -1;
  int64_t n_scalars = 0;
  const double* T_dev = sfmm_gpu_skel_device_T(skel, &skel_dev, &n_scalars);
  if (skel_dev != device)
    return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_skel: skeletons live on another device");
  const int sw = desc->kernel == SFMM_HELMHOLTZ3D || desc->kernel == SFMM_HELMHOLTZ2D ? 2 : 1;
  if (!desc->T_off || desc->n_boxes < 0 || desc->T_off[desc->n_boxes] * sw != n_scalars)
    return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_skel: descriptor T_off does not match the skeletons");
  return create_plan(desc, device, n_ranks, rank, out, T_dev, false, skel_share_T(skel));
}

int sfmm_gpu_shard_T_runs(const sfmm_plan_desc* desc, int n_ranks, int rank, int64_t* n_runs,
                          int64_t* runs, int64_t* n_entries) {
  if (!desc || !n_runs) return set_error(SFMM_EINVAL, "sfmm_gpu_shard_T_runs: null argument");
  HostPlan hp;
  std::string err;
  const int rc = build_host_plan(*desc, hp, err, n_ranks, rank);
  if (rc != SFMM_OK) return set_error(rc, err);
  *n_runs = (int64_t)hp.T_runs.size();
  if (n_entries) *n_entries = hp.T_off.empty() ? 0 : hp.T_off.back();
  if (runs)
    for (size_t i = 0; i < hp.T_runs.size(); ++i) {
      runs[2 * i] = hp.T_runs[i].src;
      runs[2 * i + 1] = hp.T_runs[i].len;
    }
  return SFMM_OK;
}

int sfmm_gpu_copy_runs(const double* src_dev, const int64_t* runs, int64_t n_runs,
                       int64_t scalars_per_entry, double* dst_dev, int device, void* stream) {
  if ((!src_dev || !dst_dev) && n_runs > 0)
    return set_error(SFMM_EINVAL, "sfmm_gpu_copy_runs: null argument");
  try {
    DeviceGuard device_guard(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t cur = 0;
    for (int64_t i = 0; i < n_runs; ++i) {
      const int64_t len = runs[2 * i + 1] * scalars_per_entry;
      ck(cudaMemcpyAsync(dst_dev + cur, src_dev + runs[2 * i] * scalars_per_entry,
                         sizeof(double) * len, cudaMemcpyDeviceToDevice, st),
         "copy runs");
      cur += len;
    }
    if (!stream) ck(cudaStreamSynchronize(st), "copy runs");  // NULL stream: complete on return
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "sfmm_gpu_copy_runs: " + f.msg);
  }
}

int sfmm_gpu_plan_create_sharded_T(const sfmm_plan_desc* desc, const void* T_owned_dev, int device,
                                   int n_ranks, int rank, sfmm_gpu_plan** out) {
  return create_plan(desc, device, n_ranks, rank, out, static_cast<const double*>(T_owned_dev),
                     true);
}

int sfmm_gpu_subtree_owners(const sfmm_tree_arrays* tree, int n_ranks, int32_t* owner) {
  if (!tree || !owner) return set_error(SFMM_EINVAL, "sfmm_gpu_subtree_owners: null argument");
  std::string err;
  const int rc = subtree_owners(tree->n_boxes, tree->level_begin, tree->depth, tree->box_parent,
                                tree->box_begin, tree->box_end, tree->box_leaf, tree->coll_off,
                                tree->coll, n_ranks, owner, err);
  return rc == SFMM_OK ? SFMM_OK : set_error(rc, err);
}

int sfmm_gpu_plan_create_sharded_owned(const sfmm_plan_desc* desc, const void* T_owned_dev,
                                       int device, int n_ranks, int rank, const int32_t* owner,
                                       sfmm_gpu_plan** out) {
  if (!owner) return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_sharded_owned: null owner");
  return create_plan(desc, device, n_ranks, rank, out, static_cast<const double*>(T_owned_dev),
                     true, {}, owner);
}

int sfmm_gpu_shard_info(const sfmm_gpu_plan* p, int64_t* send_counts, int64_t* recv_counts,
                        int64_t* n_owned_points, int64_t* n_ghost_boxes) {
  if (!p) return set_error(SFMM_EINVAL, "null plan");
  const HostPlan& hp = p->hp;
  for (int r = 0; r < hp.n_ranks; ++r) {
    const bool have = hp.send_off.size() == (size_t)hp.n_ranks + 1;
    if (send_counts) send_counts[r] = have ? hp.send_off[r + 1] - hp.send_off[r] : 0;
    if (recv_counts)
      recv_counts[r] = have ? hp.recv_off_peer[r + 1] - hp.recv_off_peer[r] : 0;
  }
  if (n_owned_points) *n_owned_points = hp.n_owned_points;
  if (n_ghost_boxes) *n_ghost_boxes = hp.n_ghost_boxes;
  return SFMM_OK;
}

int sfmm_gpu_shard_describe(const sfmm_plan_desc* desc, int n_ranks, int rank, int64_t* counts,
                            int32_t* owner, int64_t* pack_idx, int64_t* unpack_idx,
                            int32_t* owned_points) {
  if (!desc || !counts) return set_error(SFMM_EINVAL, "sfmm_gpu_shard_describe: null argument");
  HostPlan hp;
  std::string err;
  const int rc = build_host_plan(*desc, hp, err, n_ranks, rank);
  if (rc != SFMM_OK) return set_error(rc, err);
  const bool have = hp.send_off.size() == (size_t)n_ranks + 1;
  for (int r = 0; r < n_ranks; ++r) {
    counts[r] = have ? hp.send_off[r + 1] - hp.send_off[r] : 0;
    counts[n_ranks + r] = have ? hp.recv_off_peer[r + 1] - hp.recv_off_peer[r] : 0;
  }
  counts[2 * n_ranks] = hp.n_owned_points;
  counts[2 * n_ranks + 1] = hp.n_ghost_boxes;
  int64_t owned_boxes = 0;
  for (int32_t o : hp.owner) owned_boxes += o == rank ? 1 : 0;
  counts[2 * n_ranks + 2] = hp.depth < 2 ? (rank == 0 ? hp.n_boxes : 0) : owned_boxes;
  const bool have2 = hp.send2_off.size() == (size_t)n_ranks + 1;
  for (int r = 0; r < n_ranks; ++r) {
    counts[2 * n_ranks + 3 + r] = have2 ? hp.send2_off[r + 1] - hp.send2_off[r] : 0;
    counts[3 * n_ranks + 3 + r] = have2 ? hp.recv2_off[r + 1] - hp.recv2_off[r] : 0;
  }
  counts[4 * n_ranks + 3] = hp.cut_level;
  if (owner && !hp.owner.empty()) std::copy(hp.owner.begin(), hp.owner.end(), owner);
  // exchange lists in the descriptor's numbering (a compacted rank plan keeps
  // its own; the element order is the same)
  const std::vector<int64_t>& pk = hp.global_slot.empty() ? hp.pack_idx : hp.pack_idx_global;
  const std::vector<int64_t>& uk = hp.global_slot.empty() ? hp.unpack_idx : hp.unpack_idx_global;
  if (pack_idx) std::copy(pk.begin(), pk.end(), pack_idx);
  if (unpack_idx) std::copy(uk.begin(), uk.end(), unpack_idx);
  if (owned_points) {
    if (hp.depth < 2) {
      for (int64_t i = 0; i < hp.n_owned_points; ++i) owned_points[i] = (int32_t)i;
    } else {
      // owned points in slot order (as the device leaf maps order them)
      for (size_t j = 0; j < hp.leaf_box.size(); ++j) {
        const BoxRec& br = hp.box[hp.leaf_box[j]];
        for (int32_t i = 0; i < br.n; ++i)
          owned_points[hp.leaf_out[j] + hp.posmap[br.slot + i]] = desc->perm[hp.leaf_begin[j] + i];
      }
    }
  }
  return SFMM_OK;
}

int sfmm_gpu_apply_begin(sfmm_gpu_plan* p, const void* q_dev, void* send_dev, void* stream,
                         void* packed_event) {
  if (!p || !q_dev) return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->multi || p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: the plan runs its own exchange: use sfmm_gpu_apply");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    p->wait_previous(st);
    phase_begin(p, q_dev, send_dev, stream, st, static_cast<cudaEvent_t>(packed_event));
    ck(cudaGetLastError(), "kernel launch");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_apply_end(sfmm_gpu_plan* p, const void* q_dev, const void* recv_dev, void* u_dev,
                       void* stream) {
  if (!p || !u_dev) return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->multi || p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: the plan runs its own exchange: use sfmm_gpu_apply");
  if (p->dp.n_xpairs > 0 || p->dp.n_recv2 > 0)
    return set_error(SFMM_EINVAL,
                     "fmm_apply: plan has a second exchange: use sfmm_gpu_apply_mid/_fin");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    phase_end(p, q_dev, recv_dev, u_dev, stream, st);
    p->mark_done(st);
    ck(cudaGetLastError(), "kernel launch");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_apply_mid(sfmm_gpu_plan* p, const void* recv_dev, void* send2_dev, void* stream,
                       void* packed_event) {
  if (!p) return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->multi || p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: the plan runs its own exchange: use sfmm_gpu_apply");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    phase_mid(p, recv_dev, send2_dev, stream, st, static_cast<cudaEvent_t>(packed_event));
    ck(cudaGetLastError(), "kernel launch");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_apply_fin(sfmm_gpu_plan* p, const void* q_dev, const void* recv2_dev, void* u_dev,
                       void* stream) {
  if (!p || !u_dev) return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->multi || p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: the plan runs its own exchange: use sfmm_gpu_apply");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    phase_fin(p, q_dev, recv2_dev, u_dev, stream, st);
    p->mark_done(st);
    ck(cudaGetLastError(), "kernel launch");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_shard_info2(const sfmm_gpu_plan* p, int64_t* send2_counts, int64_t* recv2_counts,
                         int* cut_level) {
  if (!p) return set_error(SFMM_EINVAL, "null plan");
  const HostPlan& hp = p->hp;
  if (cut_level) *cut_level = hp.cut_level;
  for (int r = 0; r < hp.n_ranks; ++r) {
    const bool have = hp.send2_off.size() == (size_t)hp.n_ranks + 1;
    if (send2_counts) send2_counts[r] = have ? hp.send2_off[r + 1] - hp.send2_off[r] : 0;
    if (recv2_counts) recv2_counts[r] = have ? hp.recv2_off[r + 1] - hp.recv2_off[r] : 0;
  }
  return hp.xsym ? 1 : 0;
}

int sfmm_gpu_apply(sfmm_gpu_plan* p, const void* q, void* u, int nrhs, int flags,
                   sfmm_gpu_stats* stats) {
  if (!p || (!q && p->hp.n_points) || (!u && p->hp.n_points) || nrhs < 1)
    return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->hp.n_ranks > 1 && !p->multi && !p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: sharded plan without an exchange: use "
                                  "sfmm_gpu_apply_begin/_end or sfmm_gpu_plan_attach_nccl");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    const size_t col = (size_t)p->hp.n_points * p->scalar_bytes();
    const bool host = flags == SFMM_HOST_BUFFERS;
    cudaStream_t st = p->stream;
    if (host) p->ensure_io(col * nrhs);
    p->wait_previous(st);
    if (!host) {
      // device buffers: q may come from work the caller enqueued on the legacy
      // default stream, which the plan's non-blocking stream does not see
      ck(cudaEventRecord(p->ev_a, cudaStreamLegacy), "event");
      ck(cudaStreamWaitEvent(st, p->ev_a, 0), "wait caller");
    }
    ck(cudaEventRecord(p->ev_a, st), "event");
    const double* qd = static_cast<const double*>(q);
    double* ud = static_cast<double*>(u);
    if (host) {
      ck(cudaMemcpyAsync(p->io_q, q, col * nrhs, cudaMemcpyHostToDevice, st), "H2D q");
      qd = p->io_q;
      ud = p->io_u;
    }
    p->enqueue_any(qd, ud, nrhs, st, true);
    ck(cudaGetLastError(), "kernel launch");
    if (host) ck(cudaMemcpyAsync(u, p->io_u, col * nrhs, cudaMemcpyDeviceToHost, st), "D2H u");
    ck(cudaEventRecord(p->ev_b, st), "event");
    p->mark_done(st);
    ck(cudaStreamSynchronize(st), "apply");
    const int flag = multi_take_error_flag(p);
    if (stats) {
      stats->n_ifo_pairs = p->hp.n_ifo;
      stats->n_ifs_pairs = p->hp.n_ifs;
      stats->n_tfo_pairs = p->hp.n_tfo;
      stats->n_level1_pairs = p->hp.n_l1;
      stats->direct_fallback = p->hp.depth < 2 ? 1 : 0;
      if (p->hp.depth < 2) {
        stats->n_ifo_pairs = stats->n_ifs_pairs = stats->n_tfo_pairs = stats->n_level1_pairs = 0;
      }
      cudaEventElapsedTime(&stats->ms_total, p->ev_a, p->ev_b);
      stats->ms_translate = 0;
      if (p->hp.depth >= 2 && !p->multi && !p->nccl)
        cudaEventElapsedTime(&stats->ms_translate, p->ev_k2a, p->ev_k2b);
    }
    if (flag) return set_error(SFMM_EDUPLICATE, "fmm_apply: coincident points with distinct indices");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_apply_async(sfmm_gpu_plan* p, const void* q_dev, void* u_dev, int nrhs,
                         void* stream) {
  if (!p || nrhs < 1) return set_error(SFMM_EINVAL, "fmm_apply: bad arguments");
  if (p->hp.n_ranks > 1 && !p->multi && !p->nccl)
    return set_error(SFMM_EINVAL, "fmm_apply: sharded plan without an exchange: use "
                                  "sfmm_gpu_apply_begin/_end or sfmm_gpu_plan_attach_nccl");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    const double* qd = static_cast<const double*>(q_dev);
    double* ud = static_cast<double*>(u_dev);
    p->wait_previous(st);
    // Repeated applies on the same buffers replay one CUDA graph of the whole
    // sequence (~15-45 launches): launch overhead matters for small trees.
    static const bool env_graphs = [] {
      const char* v = std::getenv("SFMM_GRAPHS");
      return !(v && std::atoi(v) == 0);
    }();
    if (env_graphs && !p->timing && stream != nullptr && !p->multi && !p->nccl) {
      if (!p->graph_exec || p->graph_q != qd || p->graph_u != ud || p->graph_nrhs != nrhs) {
        if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
        p->graph_exec = nullptr;
        // device state is allocated before the capture (no cudaMalloc inside it)
        if (nrhs > 1) p->ensure_multi();
        cudaGraph_t g = nullptr;
        ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
          p->enqueue_cols(qd, ud, nrhs, st, false);
        } catch (...) {
          cudaStreamEndCapture(st, &g);  // leave the caller's stream usable
          if (g) cudaGraphDestroy(g);
          throw;
        }
        ck(cudaStreamEndCapture(st, &g), "end capture");
        ck(cudaGraphInstantiate(&p->graph_exec, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        p->graph_q = qd;
        p->graph_u = ud;
        p->graph_nrhs = nrhs;
      }
      ck(cudaGraphLaunch(p->graph_exec, st), "graph launch");
    } else {
      p->enqueue_any(qd, ud, nrhs, st, false);
    }
    p->mark_done(st);
    ck(cudaGetLastError(), "kernel launch");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, "fmm_apply: " + f.msg);
  }
}

int sfmm_gpu_check_status(sfmm_gpu_plan* p) {
  if (!p) return set_error(SFMM_EINVAL, "null plan");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    ck(cudaStreamSynchronize(p->stream), "sync");
    ck(cudaDeviceSynchronize(), "sync");
    if (multi_take_error_flag(p))
      return set_error(SFMM_EDUPLICATE, "fmm_apply: coincident points with distinct indices");
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, f.msg);
  }
}

int sfmm_gpu_plan_info_get(const sfmm_gpu_plan* p, sfmm_gpu_plan_info* info) {
  if (!p || !info) return set_error(SFMM_EINVAL, "null argument");
  const HostPlan& hp = p->hp;
  info->n_points = hp.n_points;
  info->n_boxes = hp.n_boxes;
  info->depth = hp.depth;
  info->n_slots = hp.n_slots;
  info->n_skel = hp.n_skel;
  info->m_proj = hp.m_proj;
  info->p_dense = hp.p_dense;
  info->p_skel = hp.p_skel;
  info->n_tasks = p->dp.n_tasks;
  info->device_bytes = p->device_bytes;
  info->n_ifo_pairs = hp.n_ifo;
  info->n_ifs_pairs = hp.n_ifs;
  info->n_tfo_pairs = hp.n_tfo;
  info->n_level1_pairs = hp.n_l1;
  info->sym_chain = hp.sym_chain ? 1 : 0;
  info->stage_bytes = (int64_t)(hp.stage_size * (hp.cplx ? 16 : 8));
  info->multi_sym = p->dp.multi_sym;
  info->multi_stage_bytes = p->dp.stage_m_points * kNRHS * (hp.cplx ? 16 : 8);
  info->merged_tasks = (int32_t)hp.n_merged_tasks;
  if (p->multi) {
    multi_info(p, info);  // the orchestrating plan has no level lists of its own
  } else {
    info->launches_per_apply = p->launches_per_apply();
    info->k2_grid = p->dp.k2_grid;
  }
  return SFMM_OK;
}

int sfmm_gpu_set_timing(sfmm_gpu_plan* p, int enable) {
  if (!p) return set_error(SFMM_EINVAL, "null plan");
  if (p->multi || p->nccl)
    return set_error(SFMM_EUNSUPPORTED, "set_timing: per-phase timing is per rank plan");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    if (enable && p->tev.empty()) {
      p->tev.resize((size_t)sfmm_gpu_plan::kMaxTimed * 6);
      for (cudaEvent_t& e : p->tev) ck(cudaEventCreate(&e), "cudaEventCreate");
    }
    p->timing = enable != 0;
    p->n_timed = 0;
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, f.msg);
  }
}

int sfmm_gpu_get_timings(sfmm_gpu_plan* p, float* ms, int max_applies, int* n_applies) {
  if (!p || !n_applies) return set_error(SFMM_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  try {
    DeviceGuard device_guard(p->device);
    const int n = std::min(p->n_timed, max_applies);
    for (int i = 0; i < n; ++i) {
      ck(cudaEventSynchronize(p->tev[(size_t)i * 6 + 5]), "event sync");
      for (int k = 0; k < 5; ++k)
        ck(cudaEventElapsedTime(&ms[i * 5 + k], p->tev[(size_t)i * 6 + k],
                                p->tev[(size_t)i * 6 + k + 1]),
           "event time");
    }
    *n_applies = n;
    p->n_timed = 0;
    return SFMM_OK;
  } catch (const CudaFail& f) {
    return set_error(f.code, f.msg);
  }
}

void sfmm_gpu_plan_destroy(sfmm_gpu_plan* p) { delete p; }

int sfmm_gpu_direct_sum(int kernel, double kappa, int dim, int64_t n, const double* pts,
                        const void* q, int64_t n_targets, const int32_t* targets, void* u,
                        int device) {
  if (kernel == SFMM_HELMHOLTZ2D)
    return set_error(SFMM_EUNSUPPORTED, "direct_sum_subset: helmholtz2d has no device path");
  if (n < 1 || !pts || !q || !u || n_targets < 0)
    return set_error(SFMM_EINVAL, "direct_sum_subset: bad arguments");
  for (int64_t t = 0; t < n_targets; ++t)
    if (targets[t] < 0 || targets[t] >= n)
      return set_error(SFMM_EINVAL, "direct_sum_subset: target index out of range");
  const size_t sb = kernel == SFMM_HELMHOLTZ3D ? 16 : 8;
  void *dp = nullptr, *dq = nullptr, *du = nullptr, *dt = nullptr, *de = nullptr;
  int rc = SFMM_OK;
  try {
    DeviceGuard device_guard(device);
    ck(cudaMalloc(&dp, n * dim * sizeof(double)), "cudaMalloc");
    ck(cudaMalloc(&dq, n * sb), "cudaMalloc");
    ck(cudaMalloc(&du, std::max<int64_t>(n_targets, 1) * sb), "cudaMalloc");
    ck(cudaMalloc(&dt, std::max<int64_t>(n_targets, 1) * sizeof(int32_t)), "cudaMalloc");
    ck(cudaMalloc(&de, sizeof(int)), "cudaMalloc");
    ck(cudaMemset(de, 0, sizeof(int)), "memset");
    ck(cudaMemcpy(dp, pts, n * dim * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(dq, q, n * sb, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(dt, targets, n_targets * sizeof(int32_t), cudaMemcpyHostToDevice), "H2D");
    launch_direct_subset(kernel, kappa, dim, n, (const double*)dp, (const double*)dq, n_targets,
                         (const int32_t*)dt, (double*)du, (int*)de, 0);
    ck(cudaGetLastError(), "launch");
    ck(cudaMemcpy(u, du, n_targets * sb, cudaMemcpyDeviceToHost), "D2H");
    int flag = 0;
    ck(cudaMemcpy(&flag, de, sizeof(int), cudaMemcpyDeviceToHost), "flag");
    if (flag)
      rc = set_error(SFMM_EDUPLICATE, "direct_sum_subset: coincident points with distinct indices");
  } catch (const CudaFail& f) {
    rc = set_error(f.code, "direct_sum_subset: " + f.msg);
  }
  cudaFree(dp);
  cudaFree(dq);
  cudaFree(du);
  cudaFree(dt);
  cudaFree(de);
  return rc;
}

int sfmm_gpu_plan_from_points(int kernel, double kappa, int dim, int64_t n, const double* pts,
                              int leaf_cap, double tol, double proxy_radius, int proxy_edge2d,
                              int proxy_face3d, int device, sfmm_gpu_plan** out) {
  if (!out) return set_error(SFMM_EINVAL, "plan_from_points: null argument");
  *out = nullptr;
  if (kernel == SFMM_HELMHOLTZ2D)
    return set_error(SFMM_EUNSUPPORTED, "plan_from_points: helmholtz2d has no device path");
  if (kernel < 0 || kernel > 3) return set_error(SFMM_EINVAL, "plan_from_points: bad kernel id");
  if (dim != (kernel == SFMM_LAPLACE2D ? 2 : 3))
    return set_error(SFMM_EINVAL, "plan_from_points: kernel dimension mismatch");
  if (kernel == SFMM_HELMHOLTZ3D && !(kappa > 0))
    return set_error(SFMM_EINVAL, "plan_from_points: wavenumber must be positive");
  sfmm_gpu_tree* tree = nullptr;
  int rc = sfmm_gpu_build_tree(dim, n, pts, leaf_cap, device, &tree);
  if (rc != SFMM_OK) return rc;
  sfmm_tree_arrays ta{};
  sfmm_gpu_tree_arrays(tree, &ta);
  sfmm_tree_desc td{};
  td.dim = ta.dim;
  td.n_points = ta.n_points;
  td.n_boxes = ta.n_boxes;
  td.depth = ta.depth;
  td.pts = ta.pts;
  td.level_begin = ta.level_begin;
  td.box_parent = ta.box_parent;
  td.box_level = ta.box_level;
  td.box_begin = ta.box_begin;
  td.box_end = ta.box_end;
  td.box_leaf = ta.box_leaf;
  td.box_center = ta.box_center;
  td.box_half = ta.box_half;
  sfmm_skel_result* skel = nullptr;
  rc = sfmm_gpu_build_skeletons(&td, kernel, kappa, tol, proxy_radius, proxy_edge2d, proxy_face3d,
                                device, &skel);
  if (rc == SFMM_OK) {
    sfmm_plan_desc d{};
    d.kernel = kernel;
    d.dim = dim;
    d.kappa = kappa;
    d.n_points = ta.n_points;
    d.n_boxes = ta.n_boxes;
    d.depth = ta.depth;
    d.pts = ta.pts;
    d.perm = ta.perm;
    d.level_begin = ta.level_begin;
    d.box_parent = ta.box_parent;
    d.box_level = ta.box_level;
    d.box_begin = ta.box_begin;
    d.box_end = ta.box_end;
    d.box_leaf = ta.box_leaf;
    d.coll_off = ta.coll_off;
    d.coll = ta.coll;
    d.coarse_off = ta.coarse_off;
    d.coarse = ta.coarse;
    d.fine_off = ta.fine_off;
    d.fine = ta.fine;
    // skeleton fields (T stays on the device and is copied device-to-device)
    rc = sfmm_gpu_skel_describe(skel, &d, 0, nullptr, nullptr, nullptr, nullptr);
    if (rc == SFMM_OK) rc = sfmm_gpu_plan_create_skel(&d, skel, device, 1, 0, out);
    sfmm_gpu_skel_destroy(skel);
  }
  sfmm_gpu_tree_destroy(tree);
  return rc;
}

}  // extern "C"
