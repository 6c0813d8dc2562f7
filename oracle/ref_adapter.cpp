// TEST INFRASTRUCTURE -- part of the parity oracle, never the product.
//
// extern "C" shim over the UNMODIFIED reference library, which oracle/Makefile
// compiles from /root/reference/proj/src/*.cpp into oracle/_ref/libsfmm_ref.so
// next to this file.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it.
//
// It exposes the reference's own pipeline (build_tree, build_neighbor_lists,
// build_skeletons, make_plan, fmm_apply, direct_sum_subset, the bench
// generators) and two converters:
//   * ref_desc(): reference objects  -> flat sfmm_plan_desc (include/sfmm_gpu.h)
//   * ref_from_desc(): flat descriptor -> reference Tree/NeighborLists/
//     SkeletonSet/ApplyPlan, so the reference CPU apply can run on exactly the
//     operators the GPU plan was built from.
#include <omp.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfmm/apply.hpp"
#include "sfmm/bench.hpp"
#include "sfmm/kernel.hpp"
#include "sfmm/oracle.hpp"
#include "sfmm/skeleton.hpp"
#include "sfmm/tree.hpp"
#include "sfmm_gpu.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const sfmm::DuplicatePointError& e) {
    return fail(SFMM_EDUPLICATE, e.what());
  } catch (const sfmm::DepthExceededError& e) {
    return fail(7, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(SFMM_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(9, e.what());
  }
}

struct Flat {
  std::vector<int32_t> level_begin, perm, parent, level, begin, end, poff;
  std::vector<uint8_t> leaf;
  std::vector<int64_t> iv_off, sk_off, rd_off, T_off, coll_off, coarse_off, fine_off;
  std::vector<int32_t> iv, skel_pos, red_pos, coll, coarse, fine;
  std::vector<double> T, pts;
  sfmm_plan_desc d{};
};

struct Base {
  int kernel = 0;
  double kappa = 0;
  sfmm::Tree tree;
  sfmm::NeighborLists nb;
  Flat flat;
  bool flat_ready = false;
  virtual ~Base() = default;
  virtual void apply(const void* q, void* u, int64_t* stats) = 0;
  virtual void flatten() = 0;
  virtual void info(int64_t* out) = 0;
};

template <class K>
struct Impl : Base {
  using S = typename K::scalar;
  K kern;
  sfmm::SkeletonSet<S> skel;
  sfmm::ApplyPlan<K> plan;

  void apply(const void* q, void* u, int64_t* stats) override {
    const int64_t n = tree.pts.size();
    std::vector<S> qv(reinterpret_cast<const S*>(q), reinterpret_cast<const S*>(q) + n);
    sfmm::ApplyStats st;
    std::vector<S> uv = sfmm::fmm_apply(plan, qv, &st);
    std::memcpy(u, uv.data(), sizeof(S) * n);
    if (stats) {
      stats[0] = st.n_ifo_pairs;
      stats[1] = st.n_ifs_pairs;
      stats[2] = st.n_tfo_pairs;
      stats[3] = st.n_level1_pairs;
      stats[4] = st.direct_fallback ? 1 : 0;
    }
  }

  void info(int64_t* out) override {
    out[0] = tree.depth;
    out[1] = tree.n_boxes();
    out[2] = skel.k_max;
    out[3] = skel.proj_scalars;
    out[4] = skel.saturated_boxes;
    out[5] = tree.n_leaves();
  }

  void flatten() override {
    Flat& f = flat;
    const int64_t nb_ = tree.n_boxes();
    const int d = tree.dim;
    f.level_begin = tree.level_begin;
    f.perm = tree.perm;
    f.pts = tree.pts.coords;
    f.parent.resize(nb_);
    f.level.resize(nb_);
    f.begin.resize(nb_);
    f.end.resize(nb_);
    f.poff.resize(nb_);
    f.leaf.resize(nb_);
    f.iv_off.assign(1, 0);
    f.sk_off.assign(1, 0);
    f.rd_off.assign(1, 0);
    f.T_off.assign(1, 0);
    f.coll_off.assign(1, 0);
    f.coarse_off.assign(1, 0);
    f.fine_off.assign(1, 0);
    f.iv.clear();
    f.skel_pos.clear();
    f.red_pos.clear();
    f.T.clear();
    f.coll.clear();
    f.coarse.clear();
    f.fine.clear();
    constexpr int sw = sfmm::is_complex_scalar<S>::value ? 2 : 1;
    for (int64_t b = 0; b < nb_; ++b) {
      const auto& bx = tree.boxes[b];
      // tree-only handles (ref_build_tree) have no skeletons: empty rows
      static const sfmm::BoxSkeleton<S> kNone{};
      const auto& sk = skel.box.empty() ? kNone : skel.box[b];
      f.parent[b] = bx.parent;
      f.level[b] = bx.level;
      f.begin[b] = bx.begin;
      f.end[b] = bx.end;
      f.leaf[b] = bx.leaf ? 1 : 0;
      f.poff[b] = sk.parent_offset;
      f.iv.insert(f.iv.end(), sk.index_vec.begin(), sk.index_vec.end());
      f.iv_off.push_back(static_cast<int64_t>(f.iv.size()));
      f.skel_pos.insert(f.skel_pos.end(), sk.skel_pos.begin(), sk.skel_pos.end());
      f.sk_off.push_back(static_cast<int64_t>(f.skel_pos.size()));
      f.red_pos.insert(f.red_pos.end(), sk.red_pos.begin(), sk.red_pos.end());
      f.rd_off.push_back(static_cast<int64_t>(f.red_pos.size()));
      const int64_t kr = static_cast<int64_t>(sk.skel_pos.size()) *
                         static_cast<int64_t>(sk.red_pos.size());
      if (kr > 0) {
        const double* p = reinterpret_cast<const double*>(sk.interp.data());
        f.T.insert(f.T.end(), p, p + kr * sw);
      }
      f.T_off.push_back(f.T_off.back() + kr);
      f.coll.insert(f.coll.end(), nb.colleagues[b].begin(), nb.colleagues[b].end());
      f.coll_off.push_back(static_cast<int64_t>(f.coll.size()));
      f.coarse.insert(f.coarse.end(), nb.coarse[b].begin(), nb.coarse[b].end());
      f.coarse_off.push_back(static_cast<int64_t>(f.coarse.size()));
      f.fine.insert(f.fine.end(), nb.fine[b].begin(), nb.fine[b].end());
      f.fine_off.push_back(static_cast<int64_t>(f.fine.size()));
    }
    sfmm_plan_desc& D = f.d;
    D.kernel = kernel;
    D.dim = d;
    D.kappa = kappa;
    D.n_points = tree.pts.size();
    D.n_boxes = static_cast<int32_t>(nb_);
    D.depth = tree.depth;
    D.pts = f.pts.data();
    D.perm = f.perm.data();
    D.level_begin = f.level_begin.data();
    D.box_parent = f.parent.data();
    D.box_level = f.level.data();
    D.box_begin = f.begin.data();
    D.box_end = f.end.data();
    D.box_leaf = f.leaf.data();
    D.box_parent_offset = f.poff.data();
    D.iv_off = f.iv_off.data();
    D.iv = f.iv.data();
    D.sk_off = f.sk_off.data();
    D.skel_pos = f.skel_pos.data();
    D.rd_off = f.rd_off.data();
    D.red_pos = f.red_pos.data();
    D.T_off = f.T_off.data();
    D.T = f.T.data();
    D.coll_off = f.coll_off.data();
    D.coll = f.coll.data();
    D.coarse_off = f.coarse_off.data();
    D.coarse = f.coarse.data();
    D.fine_off = f.fine_off.data();
    D.fine = f.fine.data();
    flat_ready = true;
  }
};

template <class F>
auto with_kernel(int kernel, double kappa, F&& f) {
  switch (kernel) {
    case SFMM_LAPLACE2D: return f(sfmm::Laplace2d{});
    case SFMM_LAPLACE3D: return f(sfmm::Laplace3d{});
    case SFMM_HELMHOLTZ2D: return f(sfmm::Helmholtz2d{kappa});
    case SFMM_HELMHOLTZ3D: return f(sfmm::Helmholtz3d{kappa});
  }
  throw std::invalid_argument("bad kernel id");
}

}  // namespace

extern "C" {

struct ref_handle;

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_num_threads(void) { return omp_get_max_threads(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }

int ref_generate_points(int dist, int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const auto ps = sfmm::generate_points(static_cast<sfmm::Distribution>(dist), n, seed);
    std::memcpy(out, ps.coords.data(), sizeof(double) * ps.coords.size());
  });
}

int ref_generate_charges(int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const auto q = sfmm::generate_charges(n, seed);
    std::memcpy(out, q.data(), sizeof(double) * n);
  });
}

int ref_generate_charges_complex(int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const auto q = sfmm::generate_charges_complex(n, seed);
    std::memcpy(out, q.data(), sizeof(sfmm::cplx) * n);
  });
}

// Reference pipeline: build_tree -> build_neighbor_lists -> build_skeletons ->
// make_plan (as test_apply.cpp:22-34 and bench.cpp:236-267 do).
int ref_build(int kernel, double kappa, int dim, int64_t n, const double* pts, int leaf_cap,
              double tol, double proxy_radius, int proxy_edge2d, int proxy_face3d,
              ref_handle** out) {
  return guarded([&] {
    sfmm::PointSet ps;
    ps.dim = dim;
    ps.coords.assign(pts, pts + n * dim);
    sfmm::ProxyConfig cfg;
    if (proxy_radius > 0) cfg.radius_factor = proxy_radius;
    if (proxy_edge2d > 0) cfg.edge_points_2d = proxy_edge2d;
    if (proxy_face3d > 0) cfg.face_grid_3d = proxy_face3d;
    Base* h = with_kernel(kernel, kappa, [&](auto kern) -> Base* {
      using K = decltype(kern);
      auto impl = std::make_unique<Impl<K>>();
      impl->kernel = kernel;
      impl->kappa = kappa;
      impl->kern = kern;
      impl->tree = sfmm::build_tree(ps, leaf_cap);
      impl->nb = sfmm::build_neighbor_lists(impl->tree);
      impl->skel = sfmm::build_skeletons(impl->tree, kern, tol, cfg);
      impl->plan = sfmm::make_plan(kern, impl->tree, impl->nb, impl->skel);
      return impl.release();
    });
    *out = reinterpret_cast<ref_handle*>(h);
  });
}

// Reference tree + neighbor lists only (build_tree, build_neighbor_lists):
// the descriptor's skeleton CSR is empty; apply is not available.
int ref_build_tree(int dim, int64_t n, const double* pts, int leaf_cap, ref_handle** out) {
  return guarded([&] {
    sfmm::PointSet ps;
    ps.dim = dim;
    ps.coords.assign(pts, pts + n * dim);
    auto impl = std::make_unique<Impl<sfmm::Laplace3d>>();
    impl->kernel = dim == 2 ? SFMM_LAPLACE2D : SFMM_LAPLACE3D;
    impl->tree = sfmm::build_tree(ps, leaf_cap);
    impl->nb = sfmm::build_neighbor_lists(impl->tree);
    *out = reinterpret_cast<ref_handle*>(static_cast<Base*>(impl.release()));
  });
}

// Rebuilds reference objects from a flat descriptor (any producer).
int ref_from_desc(const sfmm_plan_desc* D, ref_handle** out) {
  return guarded([&] {
    Base* h = with_kernel(D->kernel, D->kappa, [&](auto kern) -> Base* {
      using K = decltype(kern);
      using S = typename K::scalar;
      auto impl = std::make_unique<Impl<K>>();
      impl->kernel = D->kernel;
      impl->kappa = D->kappa;
      impl->kern = kern;
      sfmm::Tree& t = impl->tree;
      t.dim = D->dim;
      t.depth = D->depth;
      const int64_t n = D->n_points, nb = D->n_boxes;
      t.level_begin.assign(D->level_begin, D->level_begin + D->depth + 2);
      t.perm.assign(D->perm, D->perm + n);
      t.inv_perm.resize(n);
      for (int64_t i = 0; i < n; ++i) t.inv_perm[t.perm[i]] = static_cast<int32_t>(i);
      t.pts.dim = D->dim;
      t.pts.coords.assign(D->pts, D->pts + n * D->dim);
      t.boxes.resize(nb);
      std::vector<int> nchild(nb, 0);
      for (int64_t b = 0; b < nb; ++b) {
        auto& bx = t.boxes[b];
        bx.id = static_cast<sfmm::BoxId>(b);
        bx.parent = D->box_parent[b];
        bx.level = D->box_level[b];
        bx.begin = D->box_begin[b];
        bx.end = D->box_end[b];
        bx.leaf = D->box_leaf[b] != 0;
        if (bx.parent >= 0) t.boxes[bx.parent].child[nchild[bx.parent]++] = bx.id;
      }
      sfmm::NeighborLists& L = impl->nb;
      L.colleagues.resize(nb);
      L.coarse.resize(nb);
      L.fine.resize(nb);
      for (int64_t b = 0; b < nb; ++b) {
        L.colleagues[b].assign(D->coll + D->coll_off[b], D->coll + D->coll_off[b + 1]);
        L.coarse[b].assign(D->coarse + D->coarse_off[b], D->coarse + D->coarse_off[b + 1]);
        L.fine[b].assign(D->fine + D->fine_off[b], D->fine + D->fine_off[b + 1]);
      }
      auto& ss = impl->skel;
      ss.box.resize(nb);
      constexpr int sw = sfmm::is_complex_scalar<S>::value ? 2 : 1;
      for (int64_t b = 0; b < nb; ++b) {
        auto& sk = ss.box[b];
        sk.index_vec.assign(D->iv + D->iv_off[b], D->iv + D->iv_off[b + 1]);
        sk.skel_pos.assign(D->skel_pos + D->sk_off[b], D->skel_pos + D->sk_off[b + 1]);
        sk.red_pos.assign(D->red_pos + D->rd_off[b], D->red_pos + D->rd_off[b + 1]);
        sk.parent_offset = D->box_parent_offset[b];
        const int64_t k = static_cast<int64_t>(sk.skel_pos.size());
        const int64_t r = static_cast<int64_t>(sk.red_pos.size());
        if (D->T_off[b + 1] - D->T_off[b] != k * r)
          throw std::invalid_argument("ref_from_desc: T_off does not match k*r");
        sk.interp = sfmm::Matrix<S>(k, r);
        if (k * r > 0)
          std::memcpy(reinterpret_cast<double*>(sk.interp.data()), D->T + D->T_off[b] * sw,
                      sizeof(double) * sw * k * r);
        ss.k_max = std::max(ss.k_max, static_cast<int>(k));
        ss.proj_scalars += k * r;
      }
      impl->plan = sfmm::make_plan(kern, impl->tree, impl->nb, impl->skel);
      return impl.release();
    });
    *out = reinterpret_cast<ref_handle*>(h);
  });
}

const sfmm_plan_desc* ref_desc(ref_handle* h) {
  Base* b = reinterpret_cast<Base*>(h);
  if (!b->flat_ready) b->flatten();
  return &b->flat.d;
}

// out: depth, n_boxes, k_max, proj_scalars, saturated_boxes, n_leaves
// Box centres (n_boxes*3) and half-widths of the reference tree.
void ref_box_geometry(ref_handle* h, double* center, double* half) {
  const sfmm::Tree& t = reinterpret_cast<Base*>(h)->tree;
  for (int64_t b = 0; b < t.n_boxes(); ++b) {
    for (int k = 0; k < 3; ++k) center[3 * b + k] = t.boxes[b].center[k];
    half[b] = t.boxes[b].half;
  }
}

void ref_info(ref_handle* h, int64_t* out) { reinterpret_cast<Base*>(h)->info(out); }

// The reference CPU apply, timed by the caller.  stats: ifo, ifs, tfo, l1, fallback.
int ref_apply(ref_handle* h, const void* q, void* u, int64_t* stats) {
  return guarded([&] { reinterpret_cast<Base*>(h)->apply(q, u, stats); });
}

void ref_destroy(ref_handle* h) { delete reinterpret_cast<Base*>(h); }

// direct_sum_subset over points in their given order (oracle.cpp:51-71).
int ref_direct_sum(int kernel, double kappa, int dim, int64_t n, const double* pts,
                   const void* q, int64_t nt, const int32_t* targets, void* u) {
  return guarded([&] {
    sfmm::PointSet ps;
    ps.dim = dim;
    ps.coords.assign(pts, pts + n * dim);
    with_kernel(kernel, kappa, [&](auto kern) {
      using K = decltype(kern);
      using S = typename K::scalar;
      std::vector<S> qv(reinterpret_cast<const S*>(q), reinterpret_cast<const S*>(q) + n);
      std::vector<S> r = sfmm::direct_sum_subset(kern, ps, qv, {targets, (size_t)nt});
      std::memcpy(u, r.data(), sizeof(S) * nt);
      return 0;
    });
  });
}

// Kernel value through the reference's own eval_kernel (kernel.cpp:26-41).
int ref_eval_kernel(int kernel, double kappa, const double* x, const double* y, double* out2) {
  return guarded([&] {
    sfmm::KernelSpec spec{static_cast<sfmm::KernelFamily>(kernel), kappa};
    const int d = spec.dim();
    const sfmm::cplx g = sfmm::eval_kernel(spec, {x, (size_t)d}, {y, (size_t)d});
    out2[0] = g.real();
    out2[1] = g.imag();
  });
}

}  // extern "C"
