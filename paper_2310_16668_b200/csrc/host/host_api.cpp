// C ABI of the host descriptor container (include/sfmm_host.h) and the
// synthetic-input generators.
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "host.h"
#include "sfmm_host.h"

namespace sfmm_host {
namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

// Bit-to-double maps of the reference bench (bench.cpp:30-35).
inline double unit01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
inline double unit01_pos(std::mt19937_64& g) {
  return static_cast<double>((g() >> 11) + 1) * 0x1.0p-53;
}

// Box-Muller pairs (bench.cpp:37-45).
void normals(std::mt19937_64& g, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i += 2) {
    const double u1 = unit01_pos(g);
    const double u2 = unit01(g);
    const double rad = std::sqrt(-2.0 * std::log(u1));
    out[i] = rad * std::cos(2.0 * kPi * u2);
    if (i + 1 < n) out[i + 1] = rad * std::sin(2.0 * kPi * u2);
  }
}

}  // namespace

void generate_points(int dist, int64_t n, uint64_t seed, double* out) {
  if (n < 1) throw std::invalid_argument("generate_points: need at least one point");
  std::mt19937_64 g(seed);
  switch (dist) {
    case SFMM_DIST_SQUARE:
      for (int64_t i = 0; i < n; ++i) {
        out[2 * i] = unit01(g);
        out[2 * i + 1] = unit01(g);
      }
      break;
    case SFMM_DIST_ANNULUS:
      for (int64_t i = 0; i < n; ++i) {
        const double theta = 2.0 * kPi * unit01(g);
        const double eta = (unit01(g) - 0.5) * 0.1;
        const double r = 1.0 + 0.25 * std::cos(5.0 * theta) + eta;
        out[2 * i] = r * std::cos(theta);
        out[2 * i + 1] = r * std::sin(theta);
      }
      break;
    case SFMM_DIST_CUBE:
      for (int64_t i = 0; i < n; ++i) {
        out[3 * i] = unit01(g);
        out[3 * i + 1] = unit01(g);
        out[3 * i + 2] = unit01(g);
      }
      break;
    case SFMM_DIST_SPHERE:
      for (int64_t i = 0; i < n; ++i) {
        const double z = 2.0 * unit01(g) - 1.0;
        const double phi = 2.0 * kPi * unit01(g);
        const double s = std::sqrt(1.0 - z * z);
        out[3 * i] = s * std::cos(phi);
        out[3 * i + 1] = s * std::sin(phi);
        out[3 * i + 2] = z;
      }
      break;
    case SFMM_DIST_GAUSSIAN: {
      // Config 3(b) has no reference generator: 16 Gaussian
      // clusters, sigma 0.02, centres uniform in [0.1, 0.9]^3, all from one
      // mt19937_64 stream (centres first, then per point: cluster, 3 normals).
      double centre[16][3];
      for (auto& c : centre)
        for (double& v : c) v = 0.1 + 0.8 * unit01(g);
      for (int64_t i = 0; i < n; ++i) {
        const int c = static_cast<int>(g() % 16);
        double z[4];
        normals(g, z, 4);
        for (int k = 0; k < 3; ++k) out[3 * i + k] = centre[c][k] + 0.02 * z[k];
      }
      break;
    }
    default:
      throw std::invalid_argument("generate_points: unknown distribution");
  }
}

void generate_charges(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 g(seed);
  normals(g, out, n);
}

void generate_charges_complex(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 g(seed);
  normals(g, out, 2 * n);  // (re, im) interleaved = std::complex layout
}

}  // namespace sfmm_host

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
    return SFMM_OK;
  } catch (const std::invalid_argument& e) {
    return fail(SFMM_EINVAL, e.what());
  } catch (const std::logic_error& e) {
    return fail(SFMM_EUNSUPPORTED, e.what());
  } catch (const std::bad_alloc&) {
    return fail(SFMM_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(SFMM_EINVAL, e.what());
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct sfmm_host_plan {
  int kernel = -1;
  double kappa = 0;
  sfmm_host::Tree tree;
  sfmm_host::Neighbors nb;
  sfmm_host::Skeletons sk;
  std::vector<int32_t> parent, level, begin, end;
  std::vector<uint8_t> leaf;
  sfmm_plan_desc desc{};
  sfmm_host_info info{};

  void export_desc() {
    const int32_t n_boxes = (int32_t)tree.boxes.size();
    parent.resize(n_boxes);
    level.resize(n_boxes);
    begin.resize(n_boxes);
    end.resize(n_boxes);
    leaf.resize(n_boxes);
    for (int32_t b = 0; b < n_boxes; ++b) {
      const auto& x = tree.boxes[b];
      parent[b] = x.parent;
      level[b] = x.level;
      begin[b] = x.begin;
      end[b] = x.end;
      leaf[b] = x.leaf ? 1 : 0;
    }
    if (sk.iv_off.empty()) {  // tree only: empty skeleton CSR
      sk.iv_off.assign(n_boxes + 1, 0);
      sk.sk_off.assign(n_boxes + 1, 0);
      sk.rd_off.assign(n_boxes + 1, 0);
      sk.T_off.assign(n_boxes + 1, 0);
      sk.parent_offset.assign(n_boxes, 0);
    }
    sfmm_plan_desc& d = desc;
    d.kernel = kernel;
    d.dim = tree.dim;
    d.kappa = kappa;
    d.n_points = (int64_t)tree.perm.size();
    d.n_boxes = n_boxes;
    d.depth = tree.depth;
    d.pts = tree.pts.data();
    d.perm = tree.perm.data();
    d.level_begin = tree.level_begin.data();
    d.box_parent = parent.data();
    d.box_level = level.data();
    d.box_begin = begin.data();
    d.box_end = end.data();
    d.box_leaf = leaf.data();
    d.box_parent_offset = sk.parent_offset.data();
    d.iv_off = sk.iv_off.data();
    d.iv = sk.iv.data();
    d.sk_off = sk.sk_off.data();
    d.skel_pos = sk.skel_pos.data();
    d.rd_off = sk.rd_off.data();
    d.red_pos = sk.red_pos.data();
    d.T_off = sk.T_off.data();
    d.T = sk.T.empty() ? nullptr : sk.T.data();  // NULL: T held on the device only
    d.coll_off = nb.coll_off.data();
    d.coll = nb.coll.data();
    d.coarse_off = nb.coarse_off.data();
    d.coarse = nb.coarse.data();
    d.fine_off = nb.fine_off.data();
    d.fine = nb.fine.data();
    info.depth = tree.depth;
    info.n_boxes = n_boxes;
    info.n_leaves = 0;
    for (uint8_t l : leaf) info.n_leaves += l;
    info.k_max = sk.k_max;
    info.saturated_boxes = sk.saturated;
    info.proj_scalars = sk.proj_scalars;
  }
};

extern "C" {

const char* sfmm_host_last_error(void) { return g_err.c_str(); }

void sfmm_host_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}
int sfmm_host_get_threads(void) { return omp_get_max_threads(); }

int sfmm_host_generate_points(int dist, int64_t n, uint64_t seed, double* out) {
  return guarded([&] { sfmm_host::generate_points(dist, n, seed, out); });
}
int sfmm_host_generate_charges(int64_t n, uint64_t seed, double* out) {
  return guarded([&] { sfmm_host::generate_charges(n, seed, out); });
}
int sfmm_host_generate_charges_complex(int64_t n, uint64_t seed, double* out) {
  return guarded([&] { sfmm_host::generate_charges_complex(n, seed, out); });
}

int sfmm_host_adopt_tree(const sfmm_tree_arrays* a, sfmm_host_plan** out) {
  if (!a || !out) return fail(SFMM_EINVAL, "null argument");
  return guarded([&] {
    auto p = std::make_unique<sfmm_host_plan>();
    sfmm_host::Tree& t = p->tree;
    const int32_t nb = a->n_boxes;
    const int64_t n = a->n_points;
    t.dim = a->dim;
    t.depth = a->depth;
    t.leaf_cap = a->leaf_cap;
    t.level_begin.assign(a->level_begin, a->level_begin + a->depth + 2);
    t.perm.assign(a->perm, a->perm + n);
    t.pts.assign(a->pts, a->pts + n * a->dim);
    t.boxes.resize(nb);
    for (int32_t i = 0; i < nb; ++i) {
      sfmm_host::Box& b = t.boxes[i];
      b.parent = a->box_parent[i];
      for (int c = 0; c < 8; ++c) b.child[c] = a->box_child[8 * (int64_t)i + c];
      b.level = a->box_level[i];
      b.morton = a->box_morton[i];
      for (int k = 0; k < 3; ++k) {
        b.cell[k] = a->box_cell[3 * (int64_t)i + k];
        b.center[k] = a->box_center[3 * (int64_t)i + k];
      }
      b.half = a->box_half[i];
      b.begin = a->box_begin[i];
      b.end = a->box_end[i];
      b.leaf = a->box_leaf[i] != 0;
    }
    sfmm_host::Neighbors& g = p->nb;
    g.coll_off.assign(a->coll_off, a->coll_off + nb + 1);
    g.coll.assign(a->coll, a->coll + g.coll_off[nb]);
    g.coarse_off.assign(a->coarse_off, a->coarse_off + nb + 1);
    g.coarse.assign(a->coarse, a->coarse + g.coarse_off[nb]);
    g.fine_off.assign(a->fine_off, a->fine_off + nb + 1);
    g.fine.assign(a->fine, a->fine + g.fine_off[nb]);
    p->info.t_tree = a->seconds;
    p->export_desc();
    *out = p.release();
  });
}

const sfmm_plan_desc* sfmm_host_desc(sfmm_host_plan* p) { return p ? &p->desc : nullptr; }

int sfmm_host_box_geometry(const sfmm_host_plan* p, double* center, double* half) {
  if (!p || !center || !half) return fail(SFMM_EINVAL, "null argument");
  const auto& boxes = p->tree.boxes;
  for (size_t b = 0; b < boxes.size(); ++b) {
    for (int k = 0; k < 3; ++k) center[3 * b + k] = boxes[b].center[k];
    half[b] = boxes[b].half;
  }
  return SFMM_OK;
}

int sfmm_host_set_skeletons(sfmm_host_plan* p, const sfmm_plan_desc* s, int kernel, double kappa,
                            int32_t k_max, int64_t proj_scalars, int32_t saturated,
                            double t_skel) {
  if (!p || !s) return fail(SFMM_EINVAL, "null argument");
  return guarded([&] {
    const int64_t nb = (int64_t)p->tree.boxes.size();
    const int sw = kernel == SFMM_HELMHOLTZ3D || kernel == SFMM_HELMHOLTZ2D ? 2 : 1;
    auto& k = p->sk;
    k.iv_off.assign(s->iv_off, s->iv_off + nb + 1);
    k.sk_off.assign(s->sk_off, s->sk_off + nb + 1);
    k.rd_off.assign(s->rd_off, s->rd_off + nb + 1);
    k.T_off.assign(s->T_off, s->T_off + nb + 1);
    k.iv.assign(s->iv, s->iv + k.iv_off[nb]);
    k.skel_pos.assign(s->skel_pos, s->skel_pos + k.sk_off[nb]);
    k.red_pos.assign(s->red_pos, s->red_pos + k.rd_off[nb]);
    if (s->T)
      k.T.assign(s->T, s->T + k.T_off[nb] * sw);
    else
      std::vector<double>().swap(k.T);  // operators stay on the device (sfmm_gpu_plan_create_skel)
    k.parent_offset.assign(s->box_parent_offset, s->box_parent_offset + nb);
    k.k_max = k_max;
    k.proj_scalars = proj_scalars;
    k.saturated = saturated;
    p->kernel = kernel;
    p->kappa = kappa;
    p->info.t_skel = t_skel;
    p->export_desc();
  });
}

int sfmm_host_set_T(sfmm_host_plan* p, const double* T, int64_t n_scalars) {
  if (!p || (!T && n_scalars)) return fail(SFMM_EINVAL, "null argument");
  return guarded([&] {
    const int sw = p->kernel == SFMM_HELMHOLTZ3D || p->kernel == SFMM_HELMHOLTZ2D ? 2 : 1;
    if (p->sk.T_off.empty() || p->sk.T_off.back() * sw != n_scalars)
      throw std::invalid_argument("set_T: length does not match T_off");
    p->sk.T.assign(T, T + n_scalars);
    p->export_desc();
  });
}

int sfmm_host_info_get(const sfmm_host_plan* p, sfmm_host_info* info) {
  if (!p || !info) return fail(SFMM_EINVAL, "null argument");
  *info = p->info;
  return SFMM_OK;
}

void sfmm_host_destroy(sfmm_host_plan* p) { delete p; }

}  // extern "C"
