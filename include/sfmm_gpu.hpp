// sfmm_gpu.hpp -- header-only C++ drop-in for the reference's fmm_apply.
//
// Include AFTER the reference headers (it uses sfmm::ApplyPlan<K>,
// sfmm::ApplyStats, sfmm::DuplicatePointError from
// /root/reference/proj/include/sfmm/{apply,common}.hpp).  Usage mirrors the
// reference (README.md:127-139):
//
//     sfmm::ApplyPlan<sfmm::Laplace3d> plan = sfmm::make_plan(kern, tree, nb, skel);
//     sfmm::gpu::GpuPlan<sfmm::Laplace3d> gplan(plan);        // upload once
//     std::vector<double> u = sfmm::gpu::fmm_apply(gplan, q, &stats);
//
// The GpuPlan flattens the borrowed Tree / NeighborLists / SkeletonSet into an
// sfmm_plan_desc, uploads it to HBM and then no longer needs them.  Errors map
// back to the reference's exceptions: std::invalid_argument for size/shape
// errors (apply.cpp:313-314), sfmm::DuplicatePointError for coincident points
// with distinct ids (apply.cpp:44-46), std::runtime_error for device failures.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "sfmm_gpu.h"

namespace sfmm {
namespace gpu {

namespace detail {

inline void raise(int rc, const char* what) {
  if (rc == SFMM_OK) return;
  const std::string msg = std::string(what) + ": " + sfmm_gpu_last_error();
  if (rc == SFMM_EINVAL) throw std::invalid_argument(msg);
  if (rc == SFMM_EDUPLICATE) throw DuplicatePointError(msg);
  if (rc == SFMM_EDEPTH) throw DepthExceededError(msg);
  throw std::runtime_error(msg);
}

template <class K>
struct KernelId;
template <>
struct KernelId<Laplace2d> {
  static constexpr int value = SFMM_LAPLACE2D;
};
template <>
struct KernelId<Laplace3d> {
  static constexpr int value = SFMM_LAPLACE3D;
};
template <>
struct KernelId<Helmholtz2d> {
  static constexpr int value = SFMM_HELMHOLTZ2D;
};
template <>
struct KernelId<Helmholtz3d> {
  static constexpr int value = SFMM_HELMHOLTZ3D;
};

template <class K>
double kappa_of(const K& k) {
  if constexpr (std::is_same_v<typename K::scalar, double>)
    return 0.0;
  else
    return k.kappa;
}

template <class T, class Lists>
void flatten_lists(const Lists& lists, std::vector<int64_t>& off, std::vector<T>& flat) {
  off.assign(1, 0);
  flat.clear();
  for (const auto& l : lists) {
    flat.insert(flat.end(), l.begin(), l.end());
    off.push_back(static_cast<int64_t>(flat.size()));
  }
}

}  // namespace detail

template <class K>
class GpuPlan {
 public:
  using scalar = typename K::scalar;

  explicit GpuPlan(const ApplyPlan<K>& plan, int device = 0) : n_(plan.tree->pts.size()) {
    with_descriptor(plan, [&](const sfmm_plan_desc& d) {
      detail::raise(sfmm_gpu_plan_create(&d, device, &h_), "GpuPlan");
    });
  }

  // The same plan sharded over several GPUs of this process (whole subtrees
  // per device; ghost and column-sum exchanges by peer copies inside the
  // library, sfmm_gpu_plan_create_multi).  devices[0] holds q and u; ids may
  // repeat ({0, 0, 0, 0}: four ranks on one GPU).  fmm_apply is unchanged and
  // returns the single-GPU result.
  GpuPlan(const ApplyPlan<K>& plan, const std::vector<int>& devices) : n_(plan.tree->pts.size()) {
    if (devices.empty()) throw std::invalid_argument("GpuPlan: empty device list");
    with_descriptor(plan, [&](const sfmm_plan_desc& d) {
      detail::raise(sfmm_gpu_plan_create_multi(&d, static_cast<int>(devices.size()),
                                               devices.data(), &h_),
                    "GpuPlan");
    });
  }

 private:
  // Flattens the borrowed Tree / NeighborLists / SkeletonSet into an
  // sfmm_plan_desc (valid during the call only) and hands it to `create`.
  template <class F>
  static void with_descriptor(const ApplyPlan<K>& plan, F&& create) {
    const int64_t n = plan.tree->pts.size();
    const Tree& t = *plan.tree;
    const NeighborLists& nb = *plan.nb;
    const SkeletonSet<scalar>& sk = *plan.skel;
    const int64_t nbox = t.n_boxes();
    std::vector<int32_t> parent(nbox), level(nbox), begin(nbox), end(nbox), poff(nbox);
    std::vector<uint8_t> leaf(nbox);
    std::vector<int64_t> iv_off{0}, sk_off{0}, rd_off{0}, T_off{0}, coll_off, coarse_off, fine_off;
    std::vector<int32_t> iv, sp, rp, coll, coarse, fine;
    std::vector<double> T;
    constexpr int sw = std::is_same_v<scalar, double> ? 1 : 2;
    for (int64_t b = 0; b < nbox; ++b) {
      const TreeBox& x = t.boxes[b];
      const BoxSkeleton<scalar>& s = sk.box[b];
      parent[b] = x.parent;
      level[b] = x.level;
      begin[b] = x.begin;
      end[b] = x.end;
      leaf[b] = x.leaf ? 1 : 0;
      poff[b] = s.parent_offset;
      iv.insert(iv.end(), s.index_vec.begin(), s.index_vec.end());
      iv_off.push_back(static_cast<int64_t>(iv.size()));
      sp.insert(sp.end(), s.skel_pos.begin(), s.skel_pos.end());
      sk_off.push_back(static_cast<int64_t>(sp.size()));
      rp.insert(rp.end(), s.red_pos.begin(), s.red_pos.end());
      rd_off.push_back(static_cast<int64_t>(rp.size()));
      const int64_t kr = static_cast<int64_t>(s.skel_pos.size()) * static_cast<int64_t>(s.red_pos.size());
      const double* p = reinterpret_cast<const double*>(s.interp.data());
      if (kr) T.insert(T.end(), p, p + kr * sw);
      T_off.push_back(T_off.back() + kr);
    }
    detail::flatten_lists(nb.colleagues, coll_off, coll);
    detail::flatten_lists(nb.coarse, coarse_off, coarse);
    detail::flatten_lists(nb.fine, fine_off, fine);
    sfmm_plan_desc d{};
    d.kernel = detail::KernelId<K>::value;
    d.dim = t.dim;
    d.kappa = detail::kappa_of(plan.kernel);
    d.n_points = n;
    d.n_boxes = static_cast<int32_t>(nbox);
    d.depth = t.depth;
    d.pts = t.pts.coords.data();
    d.perm = t.perm.data();
    d.level_begin = t.level_begin.data();
    d.box_parent = parent.data();
    d.box_level = level.data();
    d.box_begin = begin.data();
    d.box_end = end.data();
    d.box_leaf = leaf.data();
    d.box_parent_offset = poff.data();
    d.iv_off = iv_off.data();
    d.iv = iv.data();
    d.sk_off = sk_off.data();
    d.skel_pos = sp.data();
    d.rd_off = rd_off.data();
    d.red_pos = rp.data();
    d.T_off = T_off.data();
    d.T = T.data();
    d.coll_off = coll_off.data();
    d.coll = coll.data();
    d.coarse_off = coarse_off.data();
    d.coarse = coarse.data();
    d.fine_off = fine_off.data();
    d.fine = fine.data();
    create(d);
  }

 public:
  // The whole pipeline on the GPU (tree, neighbor lists, skeletons, plan) from
  // the points alone -- the device counterpart of build_tree +
  // build_neighbor_lists + build_skeletons + make_plan (sfmm_gpu_plan_from_points).
  // The tree is bit-identical to the reference's; skeletons meet the same ID
  // criterion (pivots are rounding-sensitive, so not bit-identical).
  static GpuPlan from_points(const K& kernel, const PointSet& pts, int leaf_cap, double tol,
                             int device = 0) {
    GpuPlan g;
    g.n_ = pts.size();
    detail::raise(sfmm_gpu_plan_from_points(detail::KernelId<K>::value, detail::kappa_of(kernel),
                                            pts.dim, pts.size(), pts.coords.data(), leaf_cap, tol,
                                            0.0, 0, 0, device, &g.h_),
                  "GpuPlan::from_points");
    return g;
  }

  GpuPlan(GpuPlan&& o) noexcept : n_(o.n_), h_(o.h_) { o.h_ = nullptr; }
  GpuPlan(const GpuPlan&) = delete;
  GpuPlan& operator=(const GpuPlan&) = delete;
  ~GpuPlan() {
    if (h_) sfmm_gpu_plan_destroy(h_);
  }

  sfmm_gpu_plan* handle() const { return h_; }
  int64_t n_points() const { return n_; }

 private:
  GpuPlan() = default;
  int64_t n_ = 0;
  sfmm_gpu_plan* h_ = nullptr;
};

// u = A q, q and u in the original point order (apply.cpp:306-337).  Safe to
// call concurrently on one plan: applies on a plan never overlap on the device.
template <class K>
std::vector<typename K::scalar> fmm_apply(const GpuPlan<K>& plan,
                                          const std::vector<typename K::scalar>& q,
                                          ApplyStats* stats = nullptr) {
  if (static_cast<int64_t>(q.size()) != plan.n_points())
    throw std::invalid_argument("fmm_apply: charge count does not match the point count");
  std::vector<typename K::scalar> u(q.size());
  sfmm_gpu_stats st{};
  detail::raise(sfmm_gpu_apply(plan.handle(), q.data(), u.data(), 1, SFMM_HOST_BUFFERS, &st),
                "fmm_apply");
  if (stats) {
    *stats = ApplyStats{};
    stats->n_ifo_pairs = st.n_ifo_pairs;
    stats->n_ifs_pairs = st.n_ifs_pairs;
    stats->n_tfo_pairs = st.n_tfo_pairs;
    stats->n_level1_pairs = st.n_level1_pairs;
    stats->direct_fallback = st.direct_fallback != 0;
  }
  return u;
}

}  // namespace gpu
}  // namespace sfmm
