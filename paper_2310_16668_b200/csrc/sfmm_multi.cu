// Multi-GPU apply with the exchanges inside the C ABI (include/sfmm_gpu.h,
// DESIGN.md 6).  The reference is single-process (SPEC.md non-goal); its
// contract -- u in the original point order, independent of the thread count
// (apply.hpp:88-94) -- is what both paths below keep: the result is
// bit-identical to the single-GPU plan's.
//
// Ownership is whole subtrees per rank (plan_build.cpp).  One apply is
//   begin  gather + upward pass of the owned subtrees, pack the ghost boxes
//          (q slots and qhat) other ranks read              -> send
//   ghost exchange (all levels at once)                     send -> recv
//   mid    unpack, every translation task in one launch, pack the column sums
//          of the cross-rank colleague pairs this rank evaluated -> send2
//   column-sum exchange                                     send2 -> recv2
//   fin    staged + received column sums, downward pass, scatter of the owned
//          points straight into the caller's u.
//
// Two transports:
//   * MultiPlan (sfmm_gpu_plan_create_multi): ONE process drives one rank
//     plan per entry of dev_ids.  Each exchange is one cudaMemcpyPeerAsync per
//     (sender, receiver) segment over NVLink, ordered by events; q and u live
//     on the primary device and the other devices gather / scatter through
//     peer memory.  Device ids may repeat (virtual ranks on one GPU: the same
//     code path with device-local copies), which is how it is tested.
//   * NcclRank (sfmm_gpu_plan_attach_nccl): one process per GPU; the rank's
//     exchanges are grouped ncclSend/ncclRecv on the apply stream, and the
//     full result is assembled with one in-place ncclAllReduce (exact: every
//     entry has one non-zero contribution) unless SFMM_OUTPUT_OWNED.
//     libnccl is loaded at run time (dlopen), so the library has no link-time
//     NCCL dependency; a missing NCCL is SFMM_ENCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <memory>

#include "plan.h"

namespace sfmm_gpu {

namespace {

size_t scalar_doubles(const sfmm_gpu_plan* p) { return p->hp.cplx ? 2 : 1; }

// per-peer segment offsets (scalars) of one exchange, n_ranks + 1 entries
std::vector<int64_t> offsets_or_zero(const std::vector<int64_t>& v, int n) {
  if (v.size() == (size_t)n + 1) return v;
  return std::vector<int64_t>((size_t)n + 1, 0);
}

double* dev_alloc(int device, int64_t doubles, std::vector<std::pair<int, void*>>& owned) {
  DeviceGuard g(device);
  void* ptr = nullptr;
  ck(cudaMalloc(&ptr, sizeof(double) * std::max<int64_t>(doubles, 1)), "cudaMalloc(exchange)");
  owned.push_back({device, ptr});
  return static_cast<double*>(ptr);
}

}  // namespace

// ---------------------------------------------------------------------------
// single process, several devices
// ---------------------------------------------------------------------------

struct MultiRank {
  sfmm_gpu_plan* plan = nullptr;  // owned sharded rank plan
  double *send = nullptr, *recv = nullptr, *send2 = nullptr, *recv2 = nullptr;
  cudaEvent_t packed = nullptr, packed2 = nullptr, done = nullptr;
  // the ghost exchange's own stream (receiver side), so the peer copies run
  // while the rank's interior tasks do (plans split with SFMM_SHARD_OVERLAP=1)
  cudaStream_t xs = nullptr;
  cudaEvent_t xdone = nullptr;
  std::vector<int64_t> soff, roff, soff2, roff2;  // per-peer segments (scalars)
};

struct MultiPlan {
  std::vector<MultiRank> rank;
  std::vector<std::pair<int, void*>> buffers;  // (device, pointer)
  cudaEvent_t ev_in = nullptr;                 // primary: q ready / previous apply done
  bool xsym = false;                           // plans with the column-sum exchange
};

void destroy_multi(MultiPlan* m) {
  if (!m) return;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  for (MultiRank& r : m->rank) {
    if (!r.plan) continue;
    cudaSetDevice(r.plan->device);
    cudaStreamSynchronize(r.plan->stream);
    for (cudaEvent_t e : {r.packed, r.packed2, r.done, r.xdone})
      if (e) cudaEventDestroy(e);
    if (r.xs) cudaStreamDestroy(r.xs);
    delete r.plan;
  }
  for (auto& b : m->buffers) {
    cudaSetDevice(b.first);
    cudaFree(b.second);
  }
  if (m->ev_in) cudaEventDestroy(m->ev_in);
  (void)cudaGetLastError();
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

namespace {

// recv_p[roff_p[r] ..] <- send_r[soff_r[p] ..] for every ordered pair r != p
// with data: one peer copy per segment, on the receiver's stream, after the
// sender's pack.
void peer_exchange(MultiPlan& m, double* MultiRank::*send, double* MultiRank::*recv,
                   std::vector<int64_t> MultiRank::*soff, std::vector<int64_t> MultiRank::*roff,
                   cudaEvent_t MultiRank::*packed, size_t sw, bool side) {
  const int n = (int)m.rank.size();
  for (int p = 0; p < n; ++p) {
    MultiRank& dst = m.rank[p];
    DeviceGuard g(dst.plan->device);
    // the ghost exchange of a split plan runs on the receiver's exchange
    // stream, concurrently with its interior tasks; the rank stream joins it
    cudaStream_t xst = side ? dst.xs : dst.plan->stream;
    for (int r = 0; r < n; ++r) {
      if (r == p) continue;
      MultiRank& src = m.rank[r];
      const int64_t cnt = (src.*soff)[p + 1] - (src.*soff)[p];
      if (cnt == 0) continue;
      if ((dst.*roff)[r + 1] - (dst.*roff)[r] != cnt)
        throw CudaFail{SFMM_EINVAL, "exchange: peer segment sizes disagree"};
      ck(cudaStreamWaitEvent(xst, src.*packed, 0), "wait pack");
      ck(cudaMemcpyPeerAsync(dst.*recv + (dst.*roff)[r] * sw, dst.plan->device,
                             src.*send + (src.*soff)[p] * sw, src.plan->device,
                             sizeof(double) * cnt * sw, xst),
         "peer copy");
    }
    if (side) {
      ck(cudaEventRecord(dst.xdone, xst), "event");
      ck(cudaStreamWaitEvent(dst.plan->stream, dst.xdone, 0), "join exchange");
    }
  }
}

// a plan whose translation tasks are split into interior (launched before the
// ghost exchange) and boundary ones (SFMM_SHARD_OVERLAP=1)
bool split_plan(const sfmm_gpu_plan* p) {
  return p->dp.n_interior > 0 && p->dp.n_interior < p->dp.n_tasks;
}

}  // namespace

void multi_enqueue(sfmm_gpu_plan* p, const double* q, double* u, cudaStream_t st) {
  MultiPlan& m = *p->multi;
  const size_t sw = scalar_doubles(p);
  {
    DeviceGuard g(p->device);
    ck(cudaEventRecord(m.ev_in, st), "event");
  }
  for (MultiRank& r : m.rank) {
    DeviceGuard g(r.plan->device);
    cudaStream_t rs = r.plan->stream;
    ck(cudaStreamWaitEvent(rs, m.ev_in, 0), "wait input");
    phase_begin(r.plan, q, r.send, rs, rs, r.packed);
  }
  bool side = false;
  for (MultiRank& r : m.rank) side = side || split_plan(r.plan);
  peer_exchange(m, &MultiRank::send, &MultiRank::recv, &MultiRank::soff, &MultiRank::roff,
                &MultiRank::packed, sw, side);
  if (m.xsym) {
    for (MultiRank& r : m.rank) {
      DeviceGuard g(r.plan->device);
      phase_mid(r.plan, r.recv, r.send2, r.plan->stream, r.plan->stream, r.packed2);
    }
    peer_exchange(m, &MultiRank::send2, &MultiRank::recv2, &MultiRank::soff2, &MultiRank::roff2,
                  &MultiRank::packed2, sw, false);
    for (MultiRank& r : m.rank) {
      DeviceGuard g(r.plan->device);
      phase_fin(r.plan, q, r.recv2, u, r.plan->stream, r.plan->stream);
      ck(cudaEventRecord(r.done, r.plan->stream), "event");
    }
  } else {
    for (MultiRank& r : m.rank) {
      DeviceGuard g(r.plan->device);
      phase_end(r.plan, q, r.recv, u, r.plan->stream, r.plan->stream);
      ck(cudaEventRecord(r.done, r.plan->stream), "event");
    }
  }
  DeviceGuard g(p->device);
  for (MultiRank& r : m.rank) ck(cudaStreamWaitEvent(st, r.done, 0), "join ranks");
}

int multi_take_error_flag(sfmm_gpu_plan* p) {
  int any = 0;
  auto take = [&](sfmm_gpu_plan* x) {
    if (!x->dp.err_flag) return;
    DeviceGuard g(x->device);
    int flag = 0;
    ck(cudaMemcpy(&flag, x->dp.err_flag, sizeof(int), cudaMemcpyDeviceToHost), "flag");
    if (flag) {
      any = 1;
      ck(cudaMemset(x->dp.err_flag, 0, sizeof(int)), "memset");
    }
  };
  if (p->multi)
    for (MultiRank& r : p->multi->rank) take(r.plan);
  else
    take(p);
  return any;
}

void multi_info(const sfmm_gpu_plan* p, sfmm_gpu_plan_info* info) {
  info->n_tasks = 0;
  info->launches_per_apply = 0;
  for (const MultiRank& r : p->multi->rank) {
    info->n_tasks += r.plan->dp.n_tasks;
    info->launches_per_apply += r.plan->launches_per_apply();
  }
  info->k2_grid = p->multi->rank[0].plan->dp.k2_grid;
  info->sym_chain = 0;
  info->stage_bytes = 0;
  info->merged_tasks = 0;
  for (const MultiRank& r : p->multi->rank) {
    info->merged_tasks += (int32_t)r.plan->hp.n_merged_tasks;
    info->sym_chain |= r.plan->hp.sym_chain ? 1 : 0;
    info->stage_bytes += (int64_t)(r.plan->hp.stage_size * (r.plan->hp.cplx ? 16 : 8));
  }
}

namespace {

int create_multi(const sfmm_plan_desc* desc, int n_dev, const int* dev_ids, sfmm_gpu_plan** out,
                 const double* T_dev) {
  if (!desc || !out || n_dev < 1 || !dev_ids)
    return set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_multi: bad arguments");
  *out = nullptr;
  if (n_dev == 1) return create_plan(desc, dev_ids[0], 1, 0, out, T_dev, false);
  sfmm_gpu_plan* p = nullptr;
  try {
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    for (int i = 0; i < n_dev; ++i)
      if (dev_ids[i] < 0 || dev_ids[i] >= count)
        throw CudaFail{SFMM_EINVAL, "device id out of range"};
    // the other devices read q and write u on the primary, and the exchanges
    // are peer copies: every pair of distinct devices needs peer access
    for (int i = 0; i < n_dev; ++i)
      for (int j = 0; j < n_dev; ++j) {
        const int a = dev_ids[i], b = dev_ids[j];
        if (a == b) continue;
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, a, b), "cudaDeviceCanAccessPeer");
        if (!can)
          throw CudaFail{SFMM_EUNSUPPORTED, "devices " + std::to_string(a) + " and " +
                                                std::to_string(b) + " have no peer access"};
        DeviceGuard g(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer access");
        (void)cudaGetLastError();
      }
    p = new sfmm_gpu_plan();
    p->device = dev_ids[0];
    DeviceGuard g(p->device);
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreate(&p->ev_a), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_b), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_k2a), "cudaEventCreate");
    ck(cudaEventCreate(&p->ev_k2b), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(p->ev_done, p->stream), "event");
    p->multi = new MultiPlan();
    MultiPlan& m = *p->multi;
    ck(cudaEventCreateWithFlags(&m.ev_in, cudaEventDisableTiming), "cudaEventCreate");
    m.rank.resize(n_dev);
    for (int r = 0; r < n_dev; ++r) {
      const int rc = create_plan(desc, dev_ids[r], n_dev, r, &m.rank[r].plan, T_dev, false);
      if (rc != SFMM_OK) throw CudaFail{rc, sfmm_gpu_last_error()};
    }
    // the orchestrating plan mirrors the global facts of the rank plans
    const HostPlan& h0 = m.rank[0].plan->hp;
    HostPlan& hp = p->hp;
    hp.kernel = h0.kernel;
    hp.dim = h0.dim;
    hp.cplx = h0.cplx;
    hp.kappa = h0.kappa;
    hp.n_points = h0.n_points;
    hp.n_boxes = h0.n_boxes;
    hp.depth = h0.depth;
    hp.n_slots = h0.n_slots;
    hp.n_skel = h0.n_skel;
    hp.m_proj = h0.m_proj;
    hp.n_ifo = h0.n_ifo;
    hp.n_ifs = h0.n_ifs;
    hp.n_tfo = h0.n_tfo;
    hp.n_l1 = h0.n_l1;
    hp.p_dense = h0.p_dense;
    hp.p_skel = h0.p_skel;
    hp.n_ranks = n_dev;
    hp.rank = 0;
    hp.cut_level = h0.cut_level;
    hp.xsym = h0.xsym;
    m.xsym = h0.xsym;
    const size_t sw = hp.cplx ? 2 : 1;
    for (int r = 0; r < n_dev; ++r) {
      MultiRank& mr = m.rank[r];
      const HostPlan& h = mr.plan->hp;
      if (h.xsym != m.xsym) throw CudaFail{SFMM_EINVAL, "rank plans disagree on the exchanges"};
      mr.soff = offsets_or_zero(h.send_off, n_dev);
      mr.roff = offsets_or_zero(h.recv_off_peer, n_dev);
      mr.soff2 = offsets_or_zero(h.send2_off, n_dev);
      mr.roff2 = offsets_or_zero(h.recv2_off, n_dev);
      const int d = mr.plan->device;
      mr.send = dev_alloc(d, mr.soff.back() * sw, m.buffers);
      mr.recv = dev_alloc(d, mr.roff.back() * sw, m.buffers);
      mr.send2 = dev_alloc(d, mr.soff2.back() * sw, m.buffers);
      mr.recv2 = dev_alloc(d, mr.roff2.back() * sw, m.buffers);
      DeviceGuard gd(d);
      for (cudaEvent_t* e : {&mr.packed, &mr.packed2, &mr.done, &mr.xdone})
        ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaStreamCreateWithFlags(&mr.xs, cudaStreamNonBlocking), "cudaStreamCreate");
      p->device_bytes += mr.plan->device_bytes +
                         (int64_t)sizeof(double) * sw *
                             (mr.soff.back() + mr.roff.back() + mr.soff2.back() + mr.roff2.back());
    }
    *out = p;
    return SFMM_OK;
  } catch (const CudaFail& f) {
    delete p;
    return set_error(f.code, "sfmm_gpu_plan_create_multi: " + f.msg);
  } catch (const std::bad_alloc&) {
    delete p;
    return set_error(SFMM_ENOMEM, "sfmm_gpu_plan_create_multi: host allocation failed");
  }
}

// ---------------------------------------------------------------------------
// one process per GPU: NCCL, loaded at run time
// ---------------------------------------------------------------------------

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    std::vector<std::string> names;
    if (const char* env = std::getenv("SFMM_NCCL_LIB")) names.push_back(env);
    names.push_back("libnccl.so.2");
    names.push_back("libnccl.so");
    for (const std::string& n : names) {
      a.handle = dlopen(n.c_str(), RTLD_NOW | RTLD_LOCAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      a.error = "libnccl.so.2 not found (set SFMM_NCCL_LIB)";
      return a;
    }
    auto sym = [&](const char* s) { return dlsym(a.handle, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.Send || !a.Recv ||
        !a.GroupStart || !a.GroupEnd || !a.AllReduce || !a.GetErrorString) {
      a.error = "libnccl lacks a required symbol";
      a.handle = nullptr;
    }
    return a;
  }();
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw CudaFail{SFMM_ENCCL, std::string(what) + ": " + nccl_api().GetErrorString(r)};
}

}  // namespace

struct NcclRank {
  ncclComm_t comm = nullptr;
  int n_ranks = 1, rank = 0;
  // split plans (SFMM_SHARD_OVERLAP=1): the ghost exchange on its own stream,
  // concurrent with the interior tasks on the apply stream
  cudaStream_t xs = nullptr;
  cudaEvent_t packed = nullptr, xdone = nullptr;
  double *send = nullptr, *recv = nullptr, *send2 = nullptr, *recv2 = nullptr;
  std::vector<int64_t> soff, roff, soff2, roff2;
  std::vector<std::pair<int, void*>> buffers;
};

void destroy_nccl(NcclRank* n) {
  if (!n) return;
  if (n->comm && nccl_api().CommDestroy) nccl_api().CommDestroy(n->comm);
  if (n->xs) cudaStreamDestroy(n->xs);
  for (cudaEvent_t e : {n->packed, n->xdone})
    if (e) cudaEventDestroy(e);
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  for (auto& b : n->buffers) {
    cudaSetDevice(b.first);
    cudaFree(b.second);
  }
  (void)cudaGetLastError();
  if (prev >= 0) cudaSetDevice(prev);
  delete n;
}

namespace {

void nccl_exchange(NcclRank& c, const double* send, double* recv, const std::vector<int64_t>& soff,
                   const std::vector<int64_t>& roff, size_t sw, cudaStream_t st) {
  NcclApi& api = nccl_api();
  nck(api.GroupStart(), "ncclGroupStart");
  for (int peer = 0; peer < c.n_ranks; ++peer) {
    if (peer == c.rank) continue;
    const int64_t ns = soff[peer + 1] - soff[peer], nr = roff[peer + 1] - roff[peer];
    if (ns) nck(api.Send(send + soff[peer] * sw, ns * sw, ncclDouble, peer, c.comm, st), "ncclSend");
    if (nr) nck(api.Recv(recv + roff[peer] * sw, nr * sw, ncclDouble, peer, c.comm, st), "ncclRecv");
  }
  nck(api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace

void nccl_enqueue(sfmm_gpu_plan* p, const double* q, double* u, cudaStream_t st) {
  NcclRank& c = *p->nccl;
  const size_t sw = scalar_doubles(p);
  const bool full = p->output_mode == SFMM_OUTPUT_FULL;
  if (full) ck(cudaMemsetAsync(u, 0, sizeof(double) * sw * p->hp.n_points, st), "zero u");
  if (split_plan(p)) {  // exchange on the side stream while the interior tasks run
    phase_begin(p, q, c.send, st, st, c.packed);
    ck(cudaStreamWaitEvent(c.xs, c.packed, 0), "wait pack");
    nccl_exchange(c, c.send, c.recv, c.soff, c.roff, sw, c.xs);
    ck(cudaEventRecord(c.xdone, c.xs), "event");
    ck(cudaStreamWaitEvent(st, c.xdone, 0), "join exchange");
  } else {
    phase_begin(p, q, c.send, st, st, nullptr);
    nccl_exchange(c, c.send, c.recv, c.soff, c.roff, sw, st);
  }
  if (p->hp.xsym) {
    phase_mid(p, c.recv, c.send2, st, st, nullptr);
    nccl_exchange(c, c.send2, c.recv2, c.soff2, c.roff2, sw, st);
    phase_fin(p, q, c.recv2, u, st, st);
  } else {
    phase_end(p, q, c.recv, u, st, st);
  }
  if (full)
    nck(nccl_api().AllReduce(u, u, sw * p->hp.n_points, ncclDouble, ncclSum, c.comm, st),
        "ncclAllReduce");
}

}  // namespace sfmm_gpu

extern "C" {

int sfmm_gpu_plan_create_multi(const sfmm_plan_desc* desc, int n_dev, const int* dev_ids,
                               sfmm_gpu_plan** out) {
  return sfmm_gpu::create_multi(desc, n_dev, dev_ids, out, nullptr);
}

int sfmm_gpu_plan_create_multi_skel(const sfmm_plan_desc* desc, const sfmm_skel_result* skel,
                                    int n_dev, const int* dev_ids, sfmm_gpu_plan** out) {
  if (!desc || !skel || !out)
    return sfmm_gpu::set_error(SFMM_EINVAL, "sfmm_gpu_plan_create_multi_skel: null argument");
  int skel_dev = -1;
  int64_t n_scalars = 0;
  const double* T_dev = sfmm_gpu_skel_device_T(skel, &skel_dev, &n_scalars);
  const int sw = desc->kernel == SFMM_HELMHOLTZ3D || desc->kernel == SFMM_HELMHOLTZ2D ? 2 : 1;
  if (!desc->T_off || desc->n_boxes < 0 || desc->T_off[desc->n_boxes] * sw != n_scalars)
    return sfmm_gpu::set_error(
        SFMM_EINVAL, "sfmm_gpu_plan_create_multi_skel: descriptor T_off does not match the skeletons");
  return sfmm_gpu::create_multi(desc, n_dev, dev_ids, out, T_dev);
}

int sfmm_gpu_nccl_unique_id(void* id) {
  using namespace sfmm_gpu;
  if (!id) return set_error(SFMM_EINVAL, "sfmm_gpu_nccl_unique_id: null argument");
  NcclApi& api = nccl_api();
  if (!api.handle) return set_error(SFMM_ENCCL, "sfmm_gpu_nccl_unique_id: " + api.error);
  ncclUniqueId uid;
  const ncclResult_t r = api.GetUniqueId(&uid);
  if (r != ncclSuccess)
    return set_error(SFMM_ENCCL, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
  std::memcpy(id, &uid, sizeof(uid));
  return SFMM_OK;
}

int sfmm_gpu_plan_attach_nccl(sfmm_gpu_plan* p, const void* id, int n_ranks, int rank) {
  using namespace sfmm_gpu;
  if (!p || !id) return set_error(SFMM_EINVAL, "sfmm_gpu_plan_attach_nccl: null argument");
  if (p->multi || p->nccl)
    return set_error(SFMM_EINVAL, "sfmm_gpu_plan_attach_nccl: plan already has an exchange");
  if (p->hp.n_ranks != n_ranks || p->hp.rank != rank)
    return set_error(SFMM_EINVAL,
                     "sfmm_gpu_plan_attach_nccl: plan was not sharded for this rank / rank count");
  NcclApi& api = nccl_api();
  if (!api.handle) return set_error(SFMM_ENCCL, "sfmm_gpu_plan_attach_nccl: " + api.error);
  std::lock_guard<std::mutex> lock(p->mu);
  NcclRank* c = nullptr;
  try {
    DeviceGuard g(p->device);
    c = new NcclRank();
    c->n_ranks = n_ranks;
    c->rank = rank;
    const HostPlan& h = p->hp;
    const size_t sw = h.cplx ? 2 : 1;
    c->soff = offsets_or_zero(h.send_off, n_ranks);
    c->roff = offsets_or_zero(h.recv_off_peer, n_ranks);
    c->soff2 = offsets_or_zero(h.send2_off, n_ranks);
    c->roff2 = offsets_or_zero(h.recv2_off, n_ranks);
    c->send = dev_alloc(p->device, c->soff.back() * sw, c->buffers);
    c->recv = dev_alloc(p->device, c->roff.back() * sw, c->buffers);
    c->send2 = dev_alloc(p->device, c->soff2.back() * sw, c->buffers);
    c->recv2 = dev_alloc(p->device, c->roff2.back() * sw, c->buffers);
    ck(cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->packed, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&c->xdone, cudaEventDisableTiming), "cudaEventCreate");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nck(api.CommInitRank(&c->comm, n_ranks, uid, rank), "ncclCommInitRank");
    p->nccl = c;
    return SFMM_OK;
  } catch (const CudaFail& f) {
    destroy_nccl(c);
    return set_error(f.code, "sfmm_gpu_plan_attach_nccl: " + f.msg);
  }
}

int sfmm_gpu_set_output(sfmm_gpu_plan* p, int mode) {
  using namespace sfmm_gpu;
  if (!p || (mode != SFMM_OUTPUT_FULL && mode != SFMM_OUTPUT_OWNED))
    return set_error(SFMM_EINVAL, "sfmm_gpu_set_output: bad arguments");
  std::lock_guard<std::mutex> lock(p->mu);
  p->output_mode = mode;
  return SFMM_OK;
}

}  // extern "C"
