// Internal: the plan object behind the C ABI (include/sfmm_gpu.h) and the
// helpers every ABI translation unit shares (sfmm_gpu.cu, sfmm_multi.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "launch.h"
#include "plan_build.h"
#include "sfmm_gpu.h"

namespace sfmm_gpu {
int set_last_error(int code, const std::string& msg);
struct MultiPlan;  // sfmm_multi.cu: single-process multi-GPU orchestration
struct NcclRank;   // sfmm_multi.cu: NCCL exchange of a per-process rank plan
void destroy_multi(MultiPlan* m);
void destroy_nccl(NcclRank* n);
}  // namespace sfmm_gpu

namespace sfmm_gpu {

inline int set_error(int code, const std::string& msg) { return set_last_error(code, msg); }

struct CudaFail {
  int code;
  std::string msg;
};

inline void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  (void)cudaGetLastError();  // reported here; do not leak into the next call
  const int code = e == cudaErrorMemoryAllocation ? SFMM_ENOMEM : SFMM_ECUDA;
  throw CudaFail{code, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Scratch device buffers freed at scope exit.
struct TmpDev {
  std::vector<void*> ptrs;
  TmpDev() = default;
  TmpDev(const TmpDev&) = delete;
  TmpDev& operator=(const TmpDev&) = delete;
  ~TmpDev() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  const T* up(const T* src, size_t count) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    ptrs.push_back(p);
    if (count) ck(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return static_cast<const T*>(p);
  }
};

// Makes `device` current for the scope of one ABI call and restores the
// caller's device afterwards; clears stale (non-sticky) errors on entry.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ck(cudaSetDevice(device), "cudaSetDevice");
    (void)cudaGetLastError();
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace sfmm_gpu

using namespace sfmm_gpu;  // internal header: the plan below uses these unqualified

struct sfmm_gpu_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_k2a = nullptr, ev_k2b = nullptr;
  // End of the last apply enqueued on this plan (any stream).  Every apply
  // waits on it before touching the plan's shared device state (Q/U/QH/UH,
  // the column-sum staging, the task counter), so applies issued on different
  // streams -- or a sync apply on the plan stream after an async one on a
  // caller stream -- run one after another instead of racing.
  cudaEvent_t ev_done = nullptr;
  HostPlan hp;
  DevPlan dp{};
  std::vector<void*> allocs;
  std::shared_ptr<double> T_hold;  // shared operator buffer (create_plan T_share)
  int64_t device_bytes = 0;
  // per-apply state (grown on demand, one column of scalars)
  DevState ds{};
  double* io_q = nullptr;
  double* io_u = nullptr;
  size_t io_cap = 0;  // bytes of io_q / io_u
  std::mutex mu;

  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
    allocs.push_back(p);
    device_bytes += (int64_t)bytes;
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const T* src, size_t count) {
    T* d = alloc<T>(count);
    if (count) ck(cudaMemcpy(d, src, count * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return d;
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    return upload(v.data(), v.size());
  }

  // Multi-GPU.  multi: this plan drives one sharded rank plan per entry of
  // dev_ids in this process (sfmm_gpu_plan_create_multi); nccl: this sharded
  // rank plan exchanges with the other processes' ranks through NCCL
  // (sfmm_gpu_plan_attach_nccl).  Both are owned.
  MultiPlan* multi = nullptr;
  NcclRank* nccl = nullptr;
  int output_mode = SFMM_OUTPUT_FULL;

  ~sfmm_gpu_plan() {
    if (multi) destroy_multi(multi);
    if (nccl) destroy_nccl(nccl);
    int prev = -1;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : allocs) cudaFree(p);
    if (io_q) cudaFree(io_q);
    if (io_u) cudaFree(io_u);
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    if (ev_k2a) cudaEventDestroy(ev_k2a);
    if (ev_k2b) cudaEventDestroy(ev_k2b);
    if (ev_done) cudaEventDestroy(ev_done);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (PhaseGraph& g : phase_graph)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (stream) cudaStreamDestroy(stream);
    (void)cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);  // leave the caller's current device as it was
  }

  void ensure_io(size_t bytes) {
    if (bytes <= io_cap) return;
    if (io_q) cudaFree(io_q);
    if (io_u) cudaFree(io_u);
    io_q = io_u = nullptr;
    io_cap = 0;
    ck(cudaMalloc(&io_q, bytes), "cudaMalloc(q)");
    ck(cudaMalloc(&io_u, bytes), "cudaMalloc(u)");
    io_cap = bytes;
  }

  // CUDA graph of the last (q, u, nrhs) enqueued through sfmm_gpu_apply_async
  cudaGraphExec_t graph_exec = nullptr;
  const double* graph_q = nullptr;
  double* graph_u = nullptr;
  int graph_nrhs = 0;

  // Sharded applies: one CUDA graph per phase (begin, mid, fin), keyed on the
  // caller's buffers; a sequence of ~10-30 small launches per phase otherwise
  // leaves the device idle between them on deep trees.
  struct PhaseGraph {
    cudaGraphExec_t exec = nullptr;
    const void* key[3] = {nullptr, nullptr, nullptr};
  };
  PhaseGraph phase_graph[3];

  template <class F>
  void run_phase(int which, const void* k0, const void* k1, const void* k2, void* user_stream,
                 cudaStream_t st, F&& enqueue) {
    static const bool env_graphs = [] {
      const char* v = std::getenv("SFMM_GRAPHS");
      return !(v && std::atoi(v) == 0);
    }();
    if (!env_graphs || timing || user_stream == nullptr || hp.depth < 2) {
      enqueue();
      return;
    }
    PhaseGraph& g = phase_graph[which];
    if (!g.exec || g.key[0] != k0 || g.key[1] != k1 || g.key[2] != k2) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      cudaGraph_t graph = nullptr;
      ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue();
      } catch (...) {
        cudaStreamEndCapture(st, &graph);  // leave the caller's stream usable
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      ck(cudaStreamEndCapture(st, &graph), "end capture");
      ck(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
      g.key[0] = k0;
      g.key[1] = k1;
      g.key[2] = k2;
    }
    ck(cudaGraphLaunch(g.exec, st), "graph launch");
  }

  // Phase timing: 6 events per recorded apply (phase boundaries).
  static constexpr int kMaxTimed = 256;
  bool timing = false;
  std::vector<cudaEvent_t> tev;
  int n_timed = 0;

  void mark(int slot, int k, cudaStream_t st) {
    ck(cudaEventRecord(tev[(size_t)slot * 6 + k], st), "event");
  }

  // Enqueues one right-hand side: q, u device pointers in original order.
  void enqueue_one(const double* q, double* u, cudaStream_t st, bool time_k2) {
    if (hp.depth < 2) {
      launch_direct_fallback(dp, q, u, st);
      return;
    }
    const int slot = (timing && n_timed < kMaxTimed) ? n_timed++ : -1;
    if (slot >= 0) mark(slot, 0, st);
    if (dp.tree_persist) {  // one launch: the gather phase reads 0, upward holds both
      if (slot >= 0) mark(slot, 1, st);
      launch_upward_all(dp, hp, q, ds, st);
    } else {
      launch_gather(dp, q, ds, st);
      if (slot >= 0) mark(slot, 1, st);
      for (int l = hp.depth; l >= 2; --l) launch_upward(dp, hp, l, ds, st);
    }
    if (slot >= 0) mark(slot, 2, st);
    if (time_k2) ck(cudaEventRecord(ev_k2a, st), "event");
    launch_translate(dp, ds, st);
    if (time_k2) ck(cudaEventRecord(ev_k2b, st), "event");
    if (slot >= 0) mark(slot, 3, st);
    if (dp.tree_persist) {  // one launch: downward holds the scatter, which reads 0
      launch_downward_all(dp, hp, ds, u, st);
      if (slot >= 0) mark(slot, 4, st);
    } else {
      for (int l = 2; l <= hp.depth; ++l) launch_downward(dp, hp, l, ds, st);
      if (slot >= 0) mark(slot, 4, st);
      launch_scatter(dp, ds, u, st);
    }
    if (slot >= 0) mark(slot, 5, st);
  }

  // Multi-RHS state (kNRHS columns per pass), allocated on first use.
  DevState dsm{};
  bool multi_ok = true;

  void ensure_multi() {
    if (dsm.Q) return;
    const int sw = hp.cplx ? 2 : 1;
    dsm.Q = alloc<double>((size_t)hp.n_slots * kNRHS * sw);
    dsm.U = alloc<double>((size_t)hp.n_slots * kNRHS * sw);
    dsm.QH = alloc<double>((size_t)std::max<int64_t>(hp.n_skel, 1) * kNRHS * sw);
    dsm.UH = alloc<double>((size_t)std::max<int64_t>(hp.n_skel, 1) * kNRHS * sw);
    if (dp.multi_sym) {
      // staged column sums of the symmetric u pass; without the memory for
      // them the apply runs the unfolded lists instead
      void *st = nullptr, *fl = nullptr;
      const int64_t pts = std::max<int64_t>(dp.stage_m_points, kChunkM);
      const size_t bytes = (size_t)pts * kNRHS * sw * sizeof(double);
      const size_t fbytes = (size_t)(pts / kChunkM) * sizeof(unsigned);
      if (cudaMalloc(&st, bytes) == cudaSuccess && cudaMalloc(&fl, fbytes) == cudaSuccess) {
        allocs.push_back(st);
        allocs.push_back(fl);
        device_bytes += (int64_t)(bytes + fbytes);
        dsm.stage = static_cast<double*>(st);
        dsm.stage_flags = static_cast<unsigned*>(fl);
      } else {
        cudaGetLastError();
        if (st) cudaFree(st);
        dp.multi_sym = 0;
      }
    }
  }

  // nrhs columns (column-major, original order).  More than one column goes
  // through the DMMA multi-RHS passes kNRHS at a time (SFMM_MULTI=0: column
  // loop, for A/B measurements).
  void enqueue_cols(const double* q, double* u, int nrhs, cudaStream_t st, bool time_k2) {
    const size_t col_d = (size_t)hp.n_points * (hp.cplx ? 2 : 1);  // doubles per column
    static const bool env_multi = [] {
      const char* v = std::getenv("SFMM_MULTI");
      return !(v && std::atoi(v) == 0);
    }();
    if (nrhs == 1 || hp.depth < 2 || !env_multi || !dp.k2m_ok) {
      for (int r = 0; r < nrhs; ++r) enqueue_one(q + r * col_d, u + r * col_d, st, time_k2 && r == 0);
      return;
    }
    ensure_multi();
    for (int c0 = 0; c0 < nrhs; c0 += kNRHS) {
      const int nc = std::min(kNRHS, nrhs - c0);
      // phase timing records the first 16-column pass of each apply
      const int slot = (c0 == 0 && timing && n_timed < kMaxTimed) ? n_timed++ : -1;
      if (slot >= 0) mark(slot, 0, st);
      launch_gather_m(dp, q + c0 * col_d, nc, dsm, st);
      if (slot >= 0) mark(slot, 1, st);
      for (int l = hp.depth; l >= 2; --l) launch_upward_m(dp, hp, l, dsm, st);
      if (slot >= 0) mark(slot, 2, st);
      if (time_k2 && c0 == 0) ck(cudaEventRecord(ev_k2a, st), "event");
      launch_translate_m(dp, dsm, st);
      if (time_k2 && c0 == 0) ck(cudaEventRecord(ev_k2b, st), "event");
      if (slot >= 0) mark(slot, 3, st);
      for (int l = 2; l <= hp.depth; ++l) launch_downward_m(dp, hp, l, dsm, st);
      if (slot >= 0) mark(slot, 4, st);
      launch_scatter_m(dp, dsm, u + c0 * col_d, nc, st);
      if (slot >= 0) mark(slot, 5, st);
    }
  }

  // Every column of an apply: the single-GPU sequence, or one sharded apply
  // per column with the exchanges inside the library (sfmm_multi.cu).
  void enqueue_any(const double* q, double* u, int nrhs, cudaStream_t st, bool time_k2);

  int launches_per_apply() const {
    if (hp.depth < 2) return 1;
    int n = 3;  // gather, translate, scatter
    if (dp.tree_persist) {
      n = 3;  // persistent upward (with the gather), translate, persistent downward (+ scatter)
    } else {
      for (int l = 2; l <= hp.depth; ++l) {  // one launch per level and pass when both
        const bool c = hp.copy_lvl[l + 1] > hp.copy_lvl[l];  // warp boxes and items exist (k_level)
        const bool cd = hp.copy_dn_lvl[l + 1] > hp.copy_dn_lvl[l];
        const bool u = hp.up1_lvl[l + 1] > hp.up1_lvl[l], d = hp.down_lvl[l + 1] > hp.down_lvl[l];
        n += (SFMM_K1_MERGE && c && u && !dp.k1_bulk) ? 1 : (c ? 1 : 0) + (u ? 1 : 0);
        n += (SFMM_K3_MERGE && cd && d) ? 1 : (cd ? 1 : 0) + (d ? 1 : 0);
      }
    }
    if (dp.n_tasks == 0) --n;
    if (dp.n_recv > 0) ++n;  // k2b_reduce
    if (dp.leaf_pos && !dp.tree_persist) ++n;  // K4 as k4_fold + k4_gather
    // sharded plans: ghost pack / unpack, column-sum pack
    n += (dp.n_pack > 0 ? 1 : 0) + (dp.n_unpack > 0 ? 1 : 0) + (dp.n_xpairs > 0 ? 1 : 0);
    if (dp.n_interior > 0 && dp.n_interior < dp.n_tasks) ++n;  // SFMM_SHARD_OVERLAP split
    return n;
  }

  size_t scalar_bytes() const { return hp.cplx ? 16 : 8; }

  // Orders this apply after the previous one on the plan (see ev_done).
  void wait_previous(cudaStream_t st) { ck(cudaStreamWaitEvent(st, ev_done, 0), "wait previous apply"); }
  void mark_done(cudaStream_t st) { ck(cudaEventRecord(ev_done, st), "event"); }
};

namespace sfmm_gpu {

// Builds a device-resident plan (rank `rank` of `n_ranks`) on `device`.
// T_dev: the descriptor's operators in device memory (any device, global
// T_off layout), or with T_compact only the owned runs concatenated.
// T_share: owner of T_dev (a GPU skeletonization result): a single-rank plan
// whose operator layout is the descriptor's keeps the buffer instead of
// copying it (skel_share_T).
int create_plan(const sfmm_plan_desc* desc, int device, int n_ranks, int rank,
                sfmm_gpu_plan** out, const double* T_dev = nullptr, bool T_compact = false,
                std::shared_ptr<double> T_share = {}, const int32_t* l1_owner = nullptr);
std::shared_ptr<double> skel_share_T(const sfmm_skel_result* r);

// Phases of one sharded apply (sfmm_gpu.cu); throw CudaFail.
void phase_begin(sfmm_gpu_plan* p, const void* q_dev, void* send_dev, void* user_stream,
                 cudaStream_t st, cudaEvent_t packed);
void phase_mid(sfmm_gpu_plan* p, const void* recv_dev, void* send2_dev, void* user_stream,
               cudaStream_t st, cudaEvent_t packed);
void phase_fin(sfmm_gpu_plan* p, const void* q_dev, const void* recv2_dev, void* u_dev,
               void* user_stream, cudaStream_t st);
void phase_end(sfmm_gpu_plan* p, const void* q_dev, const void* recv_dev, void* u_dev,
               void* user_stream, cudaStream_t st);

// In-library exchanges (sfmm_multi.cu): one full apply of column q_dev ->
// u_dev (device buffers on p->device) enqueued on st, for a plan with
// p->multi (every rank of this process) or p->nccl (this process's rank,
// collective over the communicator).  Throw CudaFail.
void multi_enqueue(sfmm_gpu_plan* p, const double* q_dev, double* u_dev, cudaStream_t st);
void nccl_enqueue(sfmm_gpu_plan* p, const double* q_dev, double* u_dev, cudaStream_t st);
// OR of the duplicate-point flags of every rank plan (clears them).
int multi_take_error_flag(sfmm_gpu_plan* p);
// plan info of a multi-device plan: tasks, launches, bytes summed over ranks
void multi_info(const sfmm_gpu_plan* p, sfmm_gpu_plan_info* info);

}  // namespace sfmm_gpu

inline void sfmm_gpu_plan::enqueue_any(const double* q, double* u, int nrhs, cudaStream_t st,
                                       bool time_k2) {
  if (!multi && !nccl) {
    enqueue_cols(q, u, nrhs, st, time_k2);
    return;
  }
  const size_t col_d = (size_t)hp.n_points * (hp.cplx ? 2 : 1);  // doubles per column
  for (int r = 0; r < nrhs; ++r) {
    if (multi)
      sfmm_gpu::multi_enqueue(this, q + r * col_d, u + r * col_d, st);
    else
      sfmm_gpu::nccl_enqueue(this, q + r * col_d, u + r * col_d, st);
  }
}

namespace sfmm_gpu {

}  // namespace sfmm_gpu
