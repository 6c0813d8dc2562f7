// Adaptive 2:1-balanced Morton tree and its neighbor lists.
//
// Produces exactly the reference tree (/root/reference/proj/src/tree.cpp):
// identical perm, box order, point ranges, level_begin and neighbor lists.
// The construction is level-synchronous: every box of a frontier level that
// exceeds the leaf capacity is partitioned (stable, by child octant) in
// parallel, then its non-empty children are created in frontier order.  The
// balance pass must replay the reference's (level, Morton)-ordered work queue
// sequentially, because with pruned empty children the set of forced splits
// depends on the order in which they happen (tree.cpp:211-263).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <numeric>
#include <parallel/algorithm>
#include <unordered_map>

#include "host.h"

namespace sfmm_host {
namespace {

inline int octant_of(const double* x, const double* c, int dim) {
  // points on a split plane go to the upper child (tree.cpp:15-21)
  int o = 0;
  for (int k = 0; k < dim; ++k) o |= (x[k] >= c[k]) << k;
  return o;
}

inline uint64_t interleave(const int64_t* cell, int dim, int level) {
  uint64_t code = 0;
  for (int bit = 0; bit < level; ++bit)
    for (int k = 0; k < dim; ++k)
      code |= static_cast<uint64_t>((cell[k] >> bit) & 1) << (dim * bit + k);
  return code;
}

// Codes of different levels collide as integers; a leading 1 bit marks the length.
inline uint64_t level_key(int dim, int level, uint64_t code) {
  return (uint64_t{1} << (dim * level)) | code;
}

void reject_duplicates(int dim, int64_t n, const double* pts) {
  std::vector<int32_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  auto less = [&](int32_t a, int32_t b) {
    const double *pa = pts + (int64_t)a * dim, *pb = pts + (int64_t)b * dim;
    for (int k = 0; k < dim; ++k) {
      if (pa[k] < pb[k]) return true;
      if (pa[k] > pb[k]) return false;
    }
    return a < b;
  };
  __gnu_parallel::sort(ord.begin(), ord.end(), less);
  for (int64_t i = 0; i + 1 < n; ++i) {
    const double *pa = pts + (int64_t)ord[i] * dim, *pb = pts + (int64_t)ord[i + 1] * dim;
    bool same = true;
    for (int k = 0; k < dim; ++k) same = same && pa[k] == pb[k];
    if (same)
      throw DuplicatePoint("build_tree: points " + std::to_string(ord[i]) + " and " +
                           std::to_string(ord[i + 1]) + " coincide");
  }
}

class Builder {
 public:
  Builder(int dim, int64_t n, const double* pts, int leaf_cap)
      : dim_(dim), n_(n), pts_(pts), cap_(leaf_cap),
        max_depth_(dim == 2 ? kMaxDepth2 : kMaxDepth3), perm_(n), scratch_(n), oct_(n) {
    std::iota(perm_.begin(), perm_.end(), 0);
  }

  void make_root() {
    double lo[3], hi[3];
    for (int k = 0; k < dim_; ++k) {
      lo[k] = std::numeric_limits<double>::infinity();
      hi[k] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t i = 0; i < n_; ++i)
      for (int k = 0; k < dim_; ++k) {
        lo[k] = std::min(lo[k], pts_[i * dim_ + k]);
        hi[k] = std::max(hi[k], pts_[i * dim_ + k]);
      }
    Box root;
    for (int k = 0; k < dim_; ++k) {
      root.center[k] = 0.5 * (lo[k] + hi[k]);
      root.half = std::max(root.half, 0.5 * (hi[k] - lo[k]));
    }
    root.half *= 1.0 + 1e-12;  // boundary points strictly inside (tree.cpp:181-184)
    if (root.half == 0.0) root.half = 0.5;
    root.begin = 0;
    root.end = static_cast<int32_t>(n_);
    arena_.push_back(root);
    cells_.emplace(level_key(dim_, 0, 0), 0);
  }

  // Stable partition of the box's point range by child octant.
  void partition(int32_t id, int32_t counts[8]) {
    const Box& b = arena_[id];
    std::fill(counts, counts + 8, 0);
    for (int32_t i = b.begin; i < b.end; ++i) {
      const int o = octant_of(pts_ + (int64_t)perm_[i] * dim_, b.center, dim_);
      oct_[i] = static_cast<uint8_t>(o);
      ++counts[o];
    }
    int32_t pos[8];
    int32_t acc = b.begin;
    for (int c = 0; c < 8; ++c) {
      pos[c] = acc;
      acc += counts[c];
    }
    for (int32_t i = b.begin; i < b.end; ++i) scratch_[pos[oct_[i]]++] = perm_[i];
    std::memcpy(perm_.data() + b.begin, scratch_.data() + b.begin,
                sizeof(int32_t) * (size_t)(b.end - b.begin));
  }

  // Creates the non-empty children of a partitioned box (empty octants pruned).
  void make_children(int32_t id, const int32_t counts[8], std::vector<int32_t>& out) {
    arena_[id].leaf = false;
    int32_t off = arena_[id].begin;
    for (int c = 0; c < (1 << dim_); ++c) {
      if (counts[c] == 0) continue;
      const Box p = arena_[id];
      Box ch;
      ch.parent = id;
      ch.level = p.level + 1;
      ch.morton = (p.morton << dim_) | static_cast<uint64_t>(c);
      ch.half = p.half * 0.5;
      for (int k = 0; k < 3; ++k) ch.center[k] = p.center[k];
      for (int k = 0; k < dim_; ++k) {
        const int bit = (c >> k) & 1;
        ch.cell[k] = p.cell[k] * 2 + bit;
        ch.center[k] += bit ? ch.half : -ch.half;
      }
      ch.begin = off;
      ch.end = off + counts[c];
      off = ch.end;
      ch.leaf = true;
      const int32_t cid = static_cast<int32_t>(arena_.size());
      arena_.push_back(ch);
      arena_[id].child[c] = cid;
      cells_.emplace(level_key(dim_, ch.level, ch.morton), cid);
      out.push_back(cid);
    }
  }

  void split_serial(int32_t id, std::vector<int32_t>& out) {
    int32_t counts[8];
    partition(id, counts);
    make_children(id, counts, out);
  }

  void refine() {
    std::vector<int32_t> frontier{0}, next, todo;
    std::vector<std::array<int32_t, 8>> counts;
    while (!frontier.empty()) {
      todo.clear();
      for (int32_t id : frontier) {
        Box& b = arena_[id];
        if (b.npoints() <= cap_) {
          b.leaf = true;
          continue;
        }
        if (b.level == max_depth_)
          throw DepthExceeded("build_tree: leaf capacity unreachable at depth " +
                              std::to_string(max_depth_) + " (near-duplicate points?)");
        todo.push_back(id);
      }
      counts.assign(todo.size(), {});
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t t = 0; t < (int64_t)todo.size(); ++t) partition(todo[t], counts[t].data());
      next.clear();
      for (size_t t = 0; t < todo.size(); ++t) make_children(todo[t], counts[t].data(), next);
      std::swap(frontier, next);
    }
  }

  // 2:1 balance, replaying the reference work queue (tree.cpp:211-263).
  void balance() {
    std::vector<int32_t> leaves;
    for (int32_t i = 0; i < (int32_t)arena_.size(); ++i)
      if (arena_[i].leaf) leaves.push_back(i);
    std::sort(leaves.begin(), leaves.end(), [&](int32_t a, int32_t b) {
      const Box &x = arena_[a], &y = arena_[b];
      return x.level != y.level ? x.level < y.level : x.morton < y.morton;
    });
    std::deque<int32_t> work(leaves.begin(), leaves.end());
    std::vector<int32_t> created;
    const int zr = dim_ == 3 ? 1 : 0;
    while (!work.empty()) {
      const int32_t id = work.front();
      work.pop_front();
      if (!arena_[id].leaf) continue;
      for (bool again = true; again;) {
        again = false;
        const Box box = arena_[id];
        if (box.level < 2) break;
        const int64_t lim = int64_t{1} << box.level;
        for (int dz = -zr; dz <= zr; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (!dx && !dy && !dz) continue;
              const int64_t nc[3] = {box.cell[0] + dx, box.cell[1] + dy, box.cell[2] + dz};
              bool inside = true;
              for (int k = 0; k < dim_; ++k) inside = inside && nc[k] >= 0 && nc[k] < lim;
              if (!inside) continue;
              for (int lvl = box.level; lvl >= 1; --lvl) {
                const int sh = box.level - lvl;
                const int64_t cc[3] = {nc[0] >> sh, nc[1] >> sh, nc[2] >> sh};
                const auto it = cells_.find(level_key(dim_, lvl, interleave(cc, dim_, lvl)));
                if (it == cells_.end()) continue;
                const Box& cov = arena_[it->second];
                if (cov.leaf && cov.level <= box.level - 2) {
                  created.clear();
                  split_serial(it->second, created);
                  for (int32_t c : created) work.push_back(c);
                  again = true;
                }
                break;  // only the deepest covering box matters
              }
            }
      }
    }
  }

  Tree finish() {
    Tree t;
    t.dim = dim_;
    t.leaf_cap = cap_;
    const int32_t nb = static_cast<int32_t>(arena_.size());
    std::vector<int32_t> order(nb);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      const Box &x = arena_[a], &y = arena_[b];
      return x.level != y.level ? x.level < y.level : x.morton < y.morton;
    });
    std::vector<int32_t> newid(nb);
    for (int32_t i = 0; i < nb; ++i) newid[order[i]] = i;
    t.boxes.resize(nb);
    for (int32_t i = 0; i < nb; ++i) {
      Box b = arena_[order[i]];
      if (b.parent >= 0) b.parent = newid[b.parent];
      for (int32_t& c : b.child)
        if (c >= 0) c = newid[c];
      t.depth = std::max(t.depth, b.level);
      t.boxes[i] = b;
    }
    t.level_begin.assign(t.depth + 2, 0);
    for (const Box& b : t.boxes) ++t.level_begin[b.level + 1];
    for (int l = 0; l <= t.depth; ++l) t.level_begin[l + 1] += t.level_begin[l];
    t.perm = std::move(perm_);
    t.pts.resize((size_t)n_ * dim_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_; ++i)
      for (int k = 0; k < dim_; ++k) t.pts[i * dim_ + k] = pts_[(int64_t)t.perm[i] * dim_ + k];
    return t;
  }

 private:
  int dim_;
  int64_t n_;
  const double* pts_;
  int cap_, max_depth_;
  std::vector<Box> arena_;
  std::vector<int32_t> perm_, scratch_;
  std::vector<uint8_t> oct_;
  std::unordered_map<uint64_t, int32_t> cells_;
};

}  // namespace

Tree build_tree(int dim, int64_t n, const double* pts, int leaf_cap) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("build_tree: dim must be 2 or 3");
  if (leaf_cap < 1) throw std::invalid_argument("build_tree: leaf capacity must be positive");
  if (n < 1) throw std::invalid_argument("build_tree: empty point set");
  if (n > std::numeric_limits<int32_t>::max() / 2)
    throw std::invalid_argument("build_tree: point count out of range");
  for (int64_t i = 0; i < n * dim; ++i)
    if (!std::isfinite(pts[i])) throw std::invalid_argument("build_tree: non-finite coordinate");
  // SFMM_TREE_VERBOSE=1: per-phase wall time on stderr
  static const bool verbose = std::getenv("SFMM_TREE_VERBOSE") != nullptr;
  double t_prev = omp_get_wtime();
  auto mark = [&](const char* what) {
    if (!verbose) return;
    const double t = omp_get_wtime();
    std::fprintf(stderr, "[tree] %-12s %.3f s\n", what, t - t_prev);
    t_prev = t;
  };
  reject_duplicates(dim, n, pts);
  mark("duplicates");
  Builder b(dim, n, pts, leaf_cap);
  b.make_root();
  b.refine();
  mark("refine");
  b.balance();
  mark("balance");
  Tree t = b.finish();
  mark("finish");
  return t;
}

Neighbors build_neighbors(const Tree& t) {
  const int dim = t.dim;
  const int32_t nb = static_cast<int32_t>(t.boxes.size());
  std::vector<std::vector<int32_t>> coll(nb), coarse(nb), fine(nb);
  auto find = [&](int level, uint64_t code) -> int32_t {
    const Box* first = t.boxes.data() + t.level_begin[level];
    const Box* last = t.boxes.data() + t.level_begin[level + 1];
    const Box* it = std::lower_bound(first, last, code,
                                     [](const Box& b, uint64_t c) { return b.morton < c; });
    return (it != last && it->morton == code) ? static_cast<int32_t>(it - t.boxes.data()) : -1;
  };
  const int zr = dim == 3 ? 1 : 0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int32_t i = 0; i < nb; ++i) {
    const Box& b = t.boxes[i];
    const int64_t lim = int64_t{1} << b.level;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t nc[3] = {b.cell[0] + dx, b.cell[1] + dy, b.cell[2] + dz};
          bool inside = true;
          for (int k = 0; k < dim; ++k) inside = inside && nc[k] >= 0 && nc[k] < lim;
          if (!inside) continue;
          const int32_t id = find(b.level, interleave(nc, dim, b.level));
          if (id >= 0) coll[i].push_back(id);
        }
    std::sort(coll[i].begin(), coll[i].end());
  }
#pragma omp parallel for schedule(dynamic, 256)
  for (int32_t i = 0; i < nb; ++i) {
    const Box& b = t.boxes[i];
    if (b.level >= 1)
      for (int32_t c : coll[b.parent])
        if (t.boxes[c].leaf) coarse[i].push_back(c);
    if (b.leaf) {
      for (int32_t c : coll[i])
        for (int32_t g : t.boxes[c].child)
          if (g >= 0) fine[i].push_back(g);
      std::sort(fine[i].begin(), fine[i].end());
    }
  }
  Neighbors out;
  auto flatten = [nb](std::vector<std::vector<int32_t>>& lists, std::vector<int64_t>& off,
                      std::vector<int32_t>& flat) {
    off.assign(nb + 1, 0);
    for (int32_t i = 0; i < nb; ++i) off[i + 1] = off[i] + (int64_t)lists[i].size();
    flat.resize(off[nb]);
    for (int32_t i = 0; i < nb; ++i) std::copy(lists[i].begin(), lists[i].end(), flat.begin() + off[i]);
  };
  flatten(coll, out.coll_off, out.coll);
  flatten(coarse, out.coarse_off, out.coarse);
  flatten(fine, out.fine_off, out.fine);
  return out;
}

}  // namespace sfmm_host
