// Descriptor validation and flattening for the device plan (see plan_build.h).
#include "plan_build.h"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>

namespace sfmm_gpu {

namespace {

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void bad(const std::string& m) { throw Fail{SFMM_EINVAL, "sfmm_gpu_plan_create: " + m}; }

// First validation failure inside an OpenMP loop, raised after the loop.
struct ParErr {
  std::atomic<const char*> msg{nullptr};
  void set(const char* m) {
    const char* none = nullptr;
    msg.compare_exchange_strong(none, m);
  }
  void raise() const {
    if (const char* m = msg.load()) bad(m);
  }
};

}  // namespace

PlanOptions plan_options_from_env() {
  PlanOptions o;
  if (const char* v = std::getenv("SFMM_SYMMETRIC")) o.symmetric = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_SKIP_CANCEL")) o.skip_cancel = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_SHARD_OVERLAP")) o.overlap = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_SHARD_XSYM")) o.cross_symmetric = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_SYM_CHAIN")) o.sym_chain = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_MULTI_SYM")) o.multi_sym = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_TREE_PERSIST")) o.tree_persist = std::atoi(v) != 0 ? 1 : 0;
  if (const char* v = std::getenv("SFMM_SPLIT")) o.split = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_SPLIT_PART")) o.split_part = std::atof(v);
  if (const char* v = std::getenv("SFMM_SHARD_COMPACT")) o.compact = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_MERGE_TILES")) o.merge_tiles = std::atoi(v) != 0;
  if (const char* v = std::getenv("SFMM_MERGE_SHARE")) o.merge_share = std::atof(v);
  return o;
}

int subtree_owners(int32_t nb, const int32_t* level_begin, int32_t depth,
                   const int32_t* box_parent, const int32_t* box_begin, const int32_t* box_end,
                   const uint8_t* box_leaf, const int64_t* coll_off, const int32_t* coll,
                   int n_ranks, int32_t* owner, std::string& err) {
  if (nb < 1 || depth < 1 || n_ranks < 1) {
    err = "subtree_owners: bad arguments";
    return SFMM_EINVAL;
  }
  const int32_t l1b = level_begin[1], l1e = level_begin[2], n1 = l1e - l1b;
  if (n1 < n_ranks) {
    err = "subtree_owners: more ranks than level-1 subtrees";
    return SFMM_EUNSUPPORTED;
  }
  // near-field work of every leaf (its colleague leaves' points), summed per
  // level-1 subtree
  std::vector<double> cost(nb, 0.0);
  for (int32_t b = nb - 1; b >= 1; --b) {
    if (box_leaf[b]) {
      double src = 0.0;
      for (int64_t e = coll_off[b]; e < coll_off[b + 1]; ++e)
        if (box_leaf[coll[e]]) src += box_end[coll[e]] - box_begin[coll[e]];
      cost[b] += (double)(box_end[b] - box_begin[b]) * (src + 8.0);
    }
    if (box_parent[b] > 0) cost[box_parent[b]] += cost[b];
  }
  // Morton-contiguous ranges with the smallest largest cost (bisection on the
  // bound, greedy fill leaving one unit per later rank)
  double lo = 0.0, hi = 0.0;
  for (int32_t b = l1b; b < l1e; ++b) {
    lo = std::max(lo, cost[b]);
    hi += cost[b];
  }
  lo = std::max(lo, hi / n_ranks);
  auto fill = [&](double bound, bool write) {
    int r = 0;
    double acc = 0.0;
    for (int32_t b = l1b; b < l1e; ++b) {
      if (acc > 0.0 && acc + cost[b] > bound) {
        ++r;
        acc = 0.0;
      }
      if (write && acc > 0.0 && l1e - b <= n_ranks - 1 - r) {
        ++r;
        acc = 0.0;
      }
      acc += cost[b];
      if (write) owner[b] = std::min(r, n_ranks - 1);
    }
    return r + 1;
  };
  for (int it = 0; it < 60 && hi - lo > 1e-9 * hi; ++it) {
    const double mid = 0.5 * (lo + hi);
    (fill(mid, false) <= n_ranks ? hi : lo) = mid;
  }
  for (int32_t b = 0; b < l1b; ++b) owner[b] = -1;
  fill(hi, true);
  for (int32_t b = l1e; b < nb; ++b) owner[b] = owner[box_parent[b]];
  return SFMM_OK;
}

int build_host_plan(const sfmm_plan_desc& d, HostPlan& hp, std::string& err, int n_ranks,
                    int rank, int sym_chain, const int32_t* l1_owner) {
  try {
    ParErr perr;
    if (d.kernel == SFMM_HELMHOLTZ2D)
      throw Fail{SFMM_EUNSUPPORTED,
                 "sfmm_gpu_plan_create: helmholtz2d (long-double Hankel) has no device path"};
    if (d.kernel != SFMM_LAPLACE2D && d.kernel != SFMM_LAPLACE3D && d.kernel != SFMM_HELMHOLTZ3D)
      bad("unknown kernel id");
    // SFMM_PLAN_VERBOSE=1: per-phase wall time of the plan build on stderr
    static const bool verbose = std::getenv("SFMM_PLAN_VERBOSE") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto ptime = [&](const char* what) {
      if (!verbose) return;
      const auto t = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[plan] %-20s %.3f s\n", what,
                   std::chrono::duration<double>(t - t_prev).count());
      t_prev = t;
    };
    const int want_dim = d.kernel == SFMM_LAPLACE2D ? 2 : 3;
    if (d.dim != want_dim) bad("kernel dimension mismatch");  // make_plan, apply.cpp:73
    if (d.n_points < 1) bad("empty point set");
    if (d.n_boxes < 1 || d.depth < 0) bad("empty tree");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) bad("bad rank / world size");
    if (!d.pts || !d.perm || !d.level_begin || !d.box_parent || !d.box_level || !d.box_begin ||
        !d.box_end || !d.box_leaf || !d.box_parent_offset || !d.iv_off || !d.sk_off ||
        !d.rd_off || !d.T_off || !d.coll_off || !d.coarse_off || !d.fine_off)
      bad("null array in descriptor");

    hp.kernel = d.kernel;
    hp.dim = d.dim;
    hp.cplx = d.kernel == SFMM_HELMHOLTZ3D ? 1 : 0;
    hp.kappa = d.kappa;
    hp.n_points = d.n_points;
    hp.n_boxes = d.n_boxes;
    hp.depth = d.depth;
    hp.n_ranks = n_ranks;
    hp.rank = rank;
    const int64_t N = d.n_points;
    const int32_t nb = d.n_boxes;
    const int dim = d.dim;

    hp.level_begin.assign(d.level_begin, d.level_begin + d.depth + 2);
    if (hp.level_begin[0] != 0 || hp.level_begin[d.depth + 1] != nb) bad("level_begin");
    for (int l = 0; l <= d.depth; ++l)
      if (hp.level_begin[l + 1] < hp.level_begin[l]) bad("level_begin not monotone");
    for (int64_t t = 0; t < N; ++t)
      if (d.perm[t] < 0 || d.perm[t] >= N) bad("perm out of range");

    if (d.depth < 2) {
      // fmm_apply falls back to the dense sum on the original order
      // (apply.cpp:316-328); only coordinates are needed.  Sharded: rank 0
      // owns every point.
      hp.orig_pts.resize(N * dim);
      for (int64_t t = 0; t < N; ++t)
        for (int k = 0; k < dim; ++k) hp.orig_pts[(int64_t)d.perm[t] * dim + k] = d.pts[t * dim + k];
      hp.n_owned_points = rank == 0 ? N : 0;
      return SFMM_OK;
    }

    auto check_csr = [&](const int64_t* off, const int32_t* v, const char* what) {
      if (off[0] != 0) bad(std::string(what) + " offsets must start at 0");
      for (int32_t b = 0; b < nb; ++b)
        if (off[b + 1] < off[b]) bad(std::string(what) + " offsets not monotone");
      if (off[nb] > 0 && !v) bad(std::string("null ") + what);
      for (int64_t e = 0; e < off[nb]; ++e)
        if (v[e] < 0 || v[e] >= nb) bad(std::string(what) + " box id out of range");
    };
    check_csr(d.coll_off, d.coll, "colleague");
    check_csr(d.coarse_off, d.coarse, "coarse");
    check_csr(d.fine_off, d.fine, "fine");
    for (int32_t b = 0; b < nb; ++b) {
      if (d.box_parent[b] < -1 || d.box_parent[b] >= nb || (b > 0 && d.box_parent[b] < 0))
        bad("box parent out of range");
      if (b > 0 && d.box_parent[b] >= b) bad("parents must precede children (level-major order)");
    }

    ptime("validate");
    hp.box.resize(nb);
    hp.box_parent.assign(d.box_parent, d.box_parent + nb);
    hp.box_level.assign(d.box_level, d.box_level + nb);
    hp.n_slots = d.iv_off[nb];
    hp.n_skel = d.sk_off[nb];
    const int64_t S = hp.n_slots;

    // slot position map: index_vec position -> offset inside the box's slots
    hp.posmap.resize(S);
    std::vector<int32_t>& posmap = hp.posmap;
    int64_t m_proj = 0;
#pragma omp parallel reduction(+ : m_proj)
    {
      std::vector<uint8_t> seen;
#pragma omp for schedule(dynamic, 1024)
      for (int32_t b = 0; b < nb; ++b) {
        const int64_t n = d.iv_off[b + 1] - d.iv_off[b];
        const int64_t k = d.sk_off[b + 1] - d.sk_off[b];
        const int64_t r = d.rd_off[b + 1] - d.rd_off[b];
        if (n < 0 || k < 0 || r < 0) { perr.set("negative CSR extent"); continue; }
        if (!(k + r == n || (k == 0 && r == 0))) {
          perr.set("skel_pos/red_pos do not partition index_vec");
          continue;
        }
        if (d.T_off[b + 1] - d.T_off[b] != k * r) perr.set("T_off does not match k*r");
        if (d.box_level[b] < 0 || d.box_level[b] > d.depth) perr.set("box level out of range");
        BoxRec& br = hp.box[b];
        br.slot = d.iv_off[b];
        br.skel = d.sk_off[b];
        br.n = (int32_t)n;
        br.k = (int32_t)k;
        int32_t* pm = posmap.data() + d.iv_off[b];
        if (k + r == n && n > 0) {
          seen.assign(n, 0);
          for (int64_t i = 0; i < k; ++i) {
            const int32_t p = d.skel_pos[d.sk_off[b] + i];
            if (p < 0 || p >= n || seen[p]) { perr.set("skel_pos out of range or repeated"); break; }
            seen[p] = 1;
            pm[p] = (int32_t)i;
          }
          for (int64_t j = 0; j < r; ++j) {
            const int32_t p = d.red_pos[d.rd_off[b] + j];
            if (p < 0 || p >= n || seen[p]) { perr.set("red_pos out of range or repeated"); break; }
            seen[p] = 1;
            pm[p] = (int32_t)(k + j);
          }
        } else {
          for (int64_t p = 0; p < n; ++p) pm[p] = (int32_t)p;
        }
        if (d.box_leaf[b] && d.box_end[b] - d.box_begin[b] != n)
          perr.set("leaf index_vec size differs from its point range");
        m_proj += k * r;
      }
    }
    perr.raise();
    hp.m_proj = m_proj;

    ptime("posmap");
    // slot coordinates and ids are gathered on the device (every rank keeps
    // the full static geometry so ghost boxes need no remapping)
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < S; ++e)
      if (d.iv[e] < 0 || d.iv[e] >= N) perr.set("index_vec id out of range");
    perr.raise();

    ptime("slot coords");
    // upward destinations: skeleton entry i of box b lands at
    // parent position parent_offset + i (skeleton.cpp:204-218; apply.cpp:127-131)
    // (computed on the device: iv_off[p] + posmap[iv_off[p] + off + i])
    hp.parent_offset.assign(d.box_parent_offset, d.box_parent_offset + nb);
#pragma omp parallel for schedule(static)
    for (int32_t b = 0; b < nb; ++b) {
      const int32_t p = d.box_parent[b];
      const int32_t k = hp.box[b].k;
      if (k == 0) continue;
      if (p < 0) {
        perr.set("compressed root box");
        continue;
      }
      const int64_t off = d.box_parent_offset[b];
      if (off < 0 || off + k > hp.box[p].n) perr.set("parent_offset out of range");
    }
    perr.raise();

    ptime("up_dst");
    // ---- ownership: whole level-1 subtrees per rank ----------
    PlanOptions opt = plan_options_from_env();
    if (sym_chain >= 0) {  // 0 per tile, 1 chained, 2 per tile with merged tasks
      opt.sym_chain = sym_chain == 1;
      opt.merge_tiles = sym_chain == 2;
    }
    std::vector<uint8_t> unc(nb, 0);
    for (int32_t b = 0; b < nb; ++b)
      unc[b] = opt.skip_cancel && d.box_level[b] >= 2 && hp.box[b].n > 0 &&
               hp.box[b].k == hp.box[b].n;
    const int32_t l1b = hp.level_begin[1], l1e = hp.level_begin[2];
    // Sharding: each rank owns whole subtrees rooted at the cut
    // level.  Cut 1: level-1 subtrees as Morton-contiguous ranges (longest-
    // first to the least loaded rank only when the ranges cannot balance to
    // within 2 %).  Cut 2 (the level-1 split is unbalanced -- clustered
    // inputs -- or there are more ranks than level-1 boxes): level-2 subtrees
    // (and level-1 leaves) as Morton-contiguous ranges split to minimise the
    // largest estimated cost, or longest-first when a few heavy subtrees make
    // that 3 % better; the internal level-1 boxes are then shared
    // (owner kShared): every rank evaluates their level-1 translations (~0.04 %
    // of the pairs) and receives their slots, which the level-2 owners' upward
    // pass fills, with the ghosts.
    hp.owner.assign(nb, 0);
    hp.cut_level = 1;
    if (n_ranks > 1 && l1_owner) {  // given (distributed precompute): level-1 subtrees
      for (int32_t b = l1b; b < l1e; ++b) {
        if (l1_owner[b] < 0 || l1_owner[b] >= n_ranks) bad("l1_owner: rank out of range");
        hp.owner[b] = l1_owner[b];
      }
      for (int32_t b = l1e; b < nb; ++b) hp.owner[b] = hp.owner[d.box_parent[b]];
    } else if (n_ranks > 1) {
      // estimated K2 cost of every subtree, as the task cost model: lane rows
      // x (evaluated source points + 8); cancelling pairs skipped, colleague
      // blocks at ~0.575 (evaluated once for both directions)
      std::vector<double> cost(nb, 0.0);
      for (int32_t b = nb - 1; b >= 1; --b) {
        const int lev = d.box_level[b];
        double src = 0;
        if (lev >= 2) {
          for (int64_t e = d.coll_off[b]; e < d.coll_off[b + 1]; ++e) {
            const int32_t c = d.coll[e];
            if (!(unc[b] && unc[c])) src += (c == b ? 1.0 : 0.575) * hp.box[c].n;
          }
          if (!unc[b])
            for (int64_t e = d.coarse_off[b]; e < d.coarse_off[b + 1]; ++e) src += hp.box[d.coarse[e]].n;
        }
        if (lev == 1)
          for (int32_t c = l1b; c < l1e; ++c) src += hp.box[c].n;
        if (d.box_leaf[b] && lev >= 1)
          for (int64_t e = d.fine_off[b]; e < d.fine_off[b + 1]; ++e)
            if (!unc[d.fine[e]]) src += hp.box[d.fine[e]].n;
        const double lane_rows = 32.0 * ((hp.box[b].n + 31) / 32);
        cost[b] += src > 0.0 ? lane_rows * (src + 8.0) : 0.0;
        if (d.box_parent[b] > 0) cost[d.box_parent[b]] += cost[b];
      }
      const int32_t n1 = l1e - l1b;
      double total = 0.0;
      for (int32_t b = l1b; b < l1e; ++b) total += cost[b];
      const double mean = total / n_ranks;
      // Morton-contiguous split of `us` (units in Morton order) into n_ranks
      // ranges with the smallest largest estimated cost (bisection on the
      // bound, greedy fill); returns that largest cost, 1e300 if infeasible
      auto contiguous = [&](const std::vector<int32_t>& us, std::vector<int32_t>& own) {
        const int64_t nu = (int64_t)us.size();
        if (nu < n_ranks) return 1e300;
        auto fill = [&](double bound, bool write) {
          int r = 0;
          double acc = 0.0;
          for (int64_t u = 0; u < nu; ++u) {
            const double w = cost[us[u]];
            if (acc > 0.0 && acc + w > bound) {
              ++r;
              acc = 0.0;
            }
            // leave at least one unit for every later rank
            if (write && acc > 0.0 && nu - u <= n_ranks - 1 - r) {
              ++r;
              acc = 0.0;
            }
            acc += w;
            if (write) own[us[u]] = std::min(r, n_ranks - 1);
          }
          return r + 1;
        };
        double lo = mean, hi = 0.0;
        for (int32_t u : us) {
          lo = std::max(lo, cost[u]);
          hi += cost[u];
        }
        for (int it = 0; it < 60 && hi - lo > 1e-9 * hi; ++it) {
          const double mid = 0.5 * (lo + hi);
          (fill(mid, false) <= n_ranks ? hi : lo) = mid;
        }
        fill(hi, true);
        std::vector<double> load(n_ranks, 0.0);
        for (int32_t u : us) load[own[u]] += cost[u];
        return *std::max_element(load.begin(), load.end());
      };
      // longest-processing-time assignment of the same units (a few heavy
      // units: clusters); returns the largest load
      auto lpt = [&](const std::vector<int32_t>& us, std::vector<int32_t>& own) {
        if ((int64_t)us.size() < n_ranks) return 1e300;
        std::vector<int32_t> ord(us);
        std::stable_sort(ord.begin(), ord.end(),
                         [&](int32_t x, int32_t y) { return cost[x] > cost[y]; });
        std::vector<double> load(n_ranks, 0.0);
        for (int32_t u : ord) {
          const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
          own[u] = r;
          load[r] += cost[u];
        }
        return *std::max_element(load.begin(), load.end());
      };
      // cut 1: Morton-contiguous ranges of level-1 subtrees
      // whenever they balance to within 2 % of the mean (or as well as LPT),
      // else LPT
      std::vector<int32_t> l1units(n1);
      std::iota(l1units.begin(), l1units.end(), l1b);
      std::vector<int32_t> own1(nb, 0), own1_l(nb, 0);
      double max1 = contiguous(l1units, own1);
      {
        const double maxl = lpt(l1units, own1_l);
        if (max1 < 1e300 && max1 > 1.02 * mean && maxl < max1) {
          max1 = maxl;
          own1.swap(own1_l);
        }
      }
      // cut 2 units in Morton order: each level-1 box's level-2 children, or
      // the level-1 box itself when it is a leaf
      std::vector<int32_t> units;
      const int32_t l2e = d.depth >= 2 ? hp.level_begin[3] : l1e;
      {
        int32_t c = l1e;
        for (int32_t b = l1b; b < l1e; ++b) {
          if (d.box_leaf[b]) {
            units.push_back(b);
            continue;
          }
          for (; c < l2e && d.box_parent[c] == b; ++c) units.push_back(c);
        }
      }
      const int64_t nu = (int64_t)units.size();
      std::vector<int32_t> own2(nb, 0), own2_l(nb, 0);
      double max2 = contiguous(units, own2);
      if (max2 < 1e300) {
        // LPT over the same units when the contiguous ranges cannot balance;
        // the ghosts stay a small exchange
        const double maxl = lpt(units, own2_l);
        if (maxl < 0.97 * max2) {
          max2 = maxl;
          own2.swap(own2_l);
        }
      }
      if (max1 >= 1e300 && max2 >= 1e300)
        throw Fail{SFMM_EUNSUPPORTED, "sfmm_gpu_plan_create: more ranks than level-2 subtrees"};
      // cut 2 only when it clearly balances better (cut 1 has fewer ghosts)
      const bool cut2 = max1 >= 1e300 || (max2 < 1e300 && max2 < 0.95 * max1 && max1 > 1.02 * mean);
      if (verbose && rank == 0) {
        std::vector<double> l2(n_ranks, 0.0);
        if (max2 < 1e300)
          for (int32_t u : units) l2[own2[u]] += cost[u];
        double umax = 0.0;
        for (int32_t u : units) umax = std::max(umax, cost[u]);
        fprintf(stderr, "[plan] shard cost mean %.4g  cut1 max %.4g  cut2 max %.4g (%lld units, largest %.4g)  cut2 loads:",
                mean, max1, max2, (long long)nu, umax);
        for (double x : l2) fprintf(stderr, " %.3g", x);
        fprintf(stderr, "\n");
      }
      if (!cut2) {
        for (int32_t b = l1b; b < l1e; ++b) hp.owner[b] = own1[b];
      } else {
        hp.cut_level = 2;
        for (int32_t b = l1b; b < l1e; ++b) hp.owner[b] = d.box_leaf[b] ? own2[b] : kShared;
        for (int32_t b = l1e; b < l2e; ++b) hp.owner[b] = own2[b];
      }
      for (int32_t b = cut2 ? l2e : l1e; b < nb; ++b) hp.owner[b] = hp.owner[d.box_parent[b]];
    }
    auto mine = [&](int32_t b) { return hp.owner[b] == rank || hp.owner[b] == kShared; };

    ptime("ownership");
    // leaf gather/scatter maps (owned leaves): slot of position i <-> q[perm[begin + i]]
    // (apply.cpp:125, :301)
    {
      // the leaves' point ranges must tile [0, N)
      std::vector<int32_t> leaves;
      for (int32_t b = 0; b < nb; ++b)
        if (d.box_leaf[b]) leaves.push_back(b);
      {
        std::vector<std::pair<int64_t, int64_t>> rng;
        rng.reserve(leaves.size());
        for (int32_t b : leaves) rng.push_back({d.box_begin[b], d.box_end[b]});
        std::sort(rng.begin(), rng.end());
        int64_t cur = 0;
        for (auto& r : rng) {
          if (r.first != cur || r.second < r.first) {
            if (r.first < cur || r.second < r.first)
              bad("leaf point ranges overlap or exceed n_points");
            bad("leaves do not cover every point");
          }
          cur = r.second;
        }
        if (cur != N) bad(cur > N ? "leaf point ranges overlap or exceed n_points"
                                  : "leaves do not cover every point");
      }
      // owned leaves; the device scatters each one's (slot, original index)
      // pairs in slot order: position i lands at leaf_out + posmap[i]
      hp.leaf_out.assign(1, 0);
      for (int32_t b : leaves)
        if (mine(b)) {
          hp.leaf_box.push_back(b);
          hp.leaf_begin.push_back(d.box_begin[b]);
          hp.leaf_out.push_back(hp.leaf_out.back() + hp.box[b].n);
          // uncompressed leaf (k = n, level >= 2): its qhat copy / uhat fold
          // run inside K0 / K4 (the single-RHS k1_copy / k3_copy skip it)
          hp.leaf_copy.push_back(d.box_level[b] >= 2 && hp.box[b].k > 0 &&
                                 hp.box[b].k == hp.box[b].n);
        }
      hp.n_owned_points = hp.leaf_out.back();
    }

    ptime("leaf maps");
    // ---- translation entries --------------------------------------------
    //
    // Exact cancellations (in exact arithmetic) are dropped: for a box that is
    // uncompressed (level >= 2, k = n, so S = B and qhat = q) the dense add and
    // the skeleton subtract of its ifo/ifs entries cancel once the downward
    // pass adds uhat back onto u (apply.cpp:286), and a tfo entry whose source
    // is uncompressed cancels within the entry (apply.cpp:228-234).  The pair
    // counts (ApplyStats) still count them.
    //
    // With `symmetric`, an ifo pair of distinct colleagues b < c owned by the
    // same rank is evaluated once (kSYM in b's list): b's rows are accumulated
    // as usual and c's rows receive A_cb q_b = (A_bc)^T q_b as staged column
    // sums.  Pairs across ranks stay kIFO on both sides.
    hp.symmetric = opt.symmetric;
    hp.sym_chain = opt.sym_chain;
    if (hp.symmetric) {  // the colleague relation must be symmetric (and the lists sorted)
      int asym = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : asym)
      for (int32_t b = 0; b < nb; ++b)
        for (int64_t e = d.coll_off[b]; e < d.coll_off[b + 1]; ++e) {
          if (e > d.coll_off[b] && d.coll[e] <= d.coll[e - 1]) {
            asym = 1;
            break;
          }
          const int32_t c = d.coll[e];
          const int32_t* cb = d.coll + d.coll_off[c];
          const int32_t* ce = d.coll + d.coll_off[c + 1];
          if (d.box_level[c] != d.box_level[b] || !std::binary_search(cb, ce, b)) {
            asym = 1;
            break;
          }
        }
      hp.symmetric = !asym;
    }
    ptime("sym check");
    // sources(b, f): every (source, mode) evaluated for target b, before the
    // symmetric folding; identical on every rank.
    auto sources = [&](int32_t b, auto&& f) {
      const int lev = d.box_level[b];
      if (lev >= 2) {
        for (int64_t e = d.coll_off[b]; e < d.coll_off[b + 1]; ++e)
          if (!(unc[b] && unc[d.coll[e]])) f(d.coll[e], (int)kIFO);
        if (!unc[b])
          for (int64_t e = d.coarse_off[b]; e < d.coarse_off[b + 1]; ++e) f(d.coarse[e], (int)kIFS);
      }
      if (lev == 1)
        for (int32_t c = l1b; c < l1e; ++c) f(c, (int)kL1);
      if (d.box_leaf[b] && lev >= 1)
        for (int64_t e = d.fine_off[b]; e < d.fine_off[b + 1]; ++e)
          if (!unc[d.fine[e]]) f(d.fine[e], (int)kTFO);
    };

    // global pair counts and work (ApplyStats, roofline): every target
    for (int32_t b = 0; b < nb; ++b) {
      const int lev = d.box_level[b];
      auto count = [&](int32_t c, int mode) {
        const double nbn = hp.box[b].n, ncn = hp.box[c].n;
        hp.p_dense += nbn * ncn;
        if (mode == kIFO) hp.p_skel += (double)hp.box[b].k * hp.box[c].k;
        if (mode == kIFS) hp.p_skel += (double)hp.box[b].k * ncn;
        if (mode == kTFO) hp.p_skel += nbn * hp.box[c].k;
      };
      if (lev >= 2) {
        for (int64_t e = d.coll_off[b]; e < d.coll_off[b + 1]; ++e) {
          ++hp.n_ifo;
          count(d.coll[e], kIFO);
          hp.n_skipped_pairs += (unc[b] && unc[d.coll[e]]) ? 1 : 0;
        }
        for (int64_t e = d.coarse_off[b]; e < d.coarse_off[b + 1]; ++e) {
          ++hp.n_ifs;
          count(d.coarse[e], kIFS);
          hp.n_skipped_pairs += unc[b] ? 1 : 0;
        }
      }
      if (lev == 1)
        for (int32_t c = l1b; c < l1e; ++c) {
          ++hp.n_l1;
          count(c, kL1);
        }
      if (d.box_leaf[b] && lev >= 1)
        for (int64_t e = d.fine_off[b]; e < d.fine_off[b + 1]; ++e) {
          ++hp.n_tfo;
          count(d.fine[e], kTFO);
          hp.n_skipped_pairs += unc[d.fine[e]] ? 1 : 0;
        }
    }

    ptime("pair counts");
    // Cross-rank colleague pairs (xsym): each is evaluated by one of its two
    // owners.  The choice balances the ranks' estimated K2 work (dense pairs;
    // a folded pair costs ~1.15 of one direction): a greedy pass over the
    // pairs in (b < c) order gives each to the currently lighter rank.  It
    // depends only on the descriptor, so every rank derives the same choice.
    hp.xsym = hp.symmetric && n_ranks > 1 && opt.cross_symmetric;
    std::vector<uint8_t> xev;  // per colleague entry (b -> c): b's owner evaluates
    auto coll_entry = [&](int32_t b, int32_t c) {
      const int32_t* cb = d.coll + d.coll_off[b];
      const int32_t* ce = d.coll + d.coll_off[b + 1];
      return d.coll_off[b] + (int64_t)(std::lower_bound(cb, ce, c) - cb);
    };
    if (hp.xsym) {
      xev.assign(d.coll_off[nb], 0);
      std::vector<double> load(n_ranks, 0.0);
      for (int32_t b = 0; b < nb; ++b) {
        if (d.box_level[b] < 1 || hp.owner[b] == kShared) continue;
        const double nbn = hp.box[b].n;
        sources(b, [&](int32_t c, int mode) {
          if (mode == kIFO && hp.owner[c] != hp.owner[b]) return;
          const double w = (mode == kIFO && c != b) ? 0.575 : 1.0;
          load[hp.owner[b]] += w * nbn * hp.box[c].n;
        });
      }
      for (int32_t b = hp.level_begin[2]; b < nb; ++b)
        sources(b, [&](int32_t c, int mode) {
          if (mode != kIFO || c < b || hp.owner[c] == hp.owner[b]) return;
          const int rb = hp.owner[b], rc = hp.owner[c];
          const bool at_b = load[rb] <= load[rc];
          load[at_b ? rb : rc] += 1.15 * hp.box[b].n * hp.box[c].n;
          xev[coll_entry(b, c)] = at_b ? 1 : 0;
          xev[coll_entry(c, b)] = at_b ? 0 : 1;
        });
    }
    auto evaluates = [&](int32_t b, int32_t c) { return xev[coll_entry(b, c)] != 0; };
    // cross-rank colleague pair (b, c) that b's owner does not evaluate
    auto folded_away = [&](int32_t b, int32_t c, int mode) {
      return hp.xsym && mode == kIFO && hp.owner[b] != hp.owner[c] && !evaluates(b, c);
    };
    // Compact slot space (sharded plans): only the boxes this rank touches --
    // its own (and shared) boxes and the sources its targets read -- keep
    // slots, renumbered into one contiguous range, so the slot geometry and
    // state (coordinates, ids, Q / U, QH / UH: ~50 B per slot) scale with the
    // rank's share instead of N.  Every other box gets slot = skel = -1 and is
    // never touched.  Slot offsets are only reached through the box records,
    // the exchange index lists and the leaf maps, all built from here on.
    hp.global_slot.clear();
    if (n_ranks > 1 && opt.compact) {
      std::vector<uint8_t> present(nb, 0);
      for (int32_t b = 0; b < nb; ++b) {
        if (!mine(b)) continue;
        present[b] = 1;
        if (d.box_level[b] >= 1) sources(b, [&](int32_t c, int) { present[c] = 1; });
      }
      std::vector<int32_t> pm;
      int64_t cs = 0, ck = 0;
      hp.global_slot.assign(nb, -1);
      hp.global_skel.assign(nb, -1);
      for (int32_t b = 0; b < nb; ++b) {
        BoxRec& br = hp.box[b];
        hp.global_slot[b] = br.slot;
        hp.global_skel[b] = br.skel;
        if (!present[b]) {
          br.slot = -1;
          br.skel = -1;
          continue;
        }
        pm.insert(pm.end(), hp.posmap.begin() + br.slot, hp.posmap.begin() + br.slot + br.n);
        hp.iv_runs.push_back({br.slot, cs, br.n});
        br.slot = cs;
        br.skel = ck;
        cs += br.n;
        ck += br.k;
      }
      hp.posmap.swap(pm);
      hp.n_slots = cs;
      hp.n_skel = ck;
    }
    // this rank's CSR: owned targets only
    hp.ent_range.resize(nb);
    std::vector<uint8_t> boundary(nb, 0);
    for (int32_t b = 0; b < nb; ++b) {
      EntryRange& er = hp.ent_range[b];
      er.begin = (int64_t)hp.entries.size();
      er.count = 0;
      if (!mine(b) || d.box_level[b] < 1) continue;
      sources(b, [&](int32_t c, int mode) {
        if (mode == kIFO && hp.xsym && !mine(c)) {
          if (evaluates(b, c)) {  // evaluated here; c's side goes back to its owner
            hp.entries.push_back((c << kModeBits) | kSYM);
            boundary[b] = 1;
          }
          return;  // otherwise c's owner evaluates it and sends b's column sums
        }
        if (!mine(c)) boundary[b] = 1;
        if (mode == kIFO && hp.symmetric && c != b && mine(c)) {
          if (c > b) hp.entries.push_back((c << kModeBits) | kSYM);
          return;  // c < b arrives through c's staged column sums
        }
        hp.entries.push_back((c << kModeBits) | mode);
        hp.p_dense_local += (double)hp.box[b].n * hp.box[c].n;
      });
      er.count = (int32_t)((int64_t)hp.entries.size() - er.begin);
      for (int64_t e = er.begin; e < er.begin + er.count; ++e)
        if ((hp.entries[e] & kModeMask) == kSYM)
          hp.p_dense_local += (double)hp.box[b].n * hp.box[hp.entries[e] >> kModeBits].n;
    }

    ptime("csr");
    // multi-RHS path: the same entries without the symmetric folding, and
    // 16-row tasks (cost sorted, interior first is not needed: the multi-RHS
    // apply is single-rank)
    {
      hp.ent_range_full.resize(nb);
      std::vector<std::pair<double, Task>> tv;
      std::vector<std::pair<double, Task>> th;  // the uhat pass: its own costs
      for (int32_t b = 0; b < nb; ++b) {
        EntryRange& er = hp.ent_range_full[b];
        er.begin = (int64_t)hp.entries_full.size();
        er.count = 0;
        if (!mine(b) || d.box_level[b] < 1) continue;
        double src = 0, hsrc = 0;
        sources(b, [&](int32_t c, int mode) {
          hp.entries_full.push_back((c << kModeBits) | mode);
          src += hp.box[c].n;
          hsrc += mode == kIFS ? hp.box[c].n : (mode == kIFO ? hp.box[c].k : 0);
        });
        er.count = (int32_t)((int64_t)hp.entries_full.size() - er.begin);
        if (er.count == 0) continue;
        for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += kMultiRows) {
          const Task t{b, r0, std::min(kMultiRows, hp.box[b].n - r0), 0, 0};
          tv.push_back({src * kMultiRows + 64.0, t});
          if (r0 < hp.box[b].k) {  // skeleton rows (16-row warp granularity) x h-weighted sources
            const int32_t hr = std::min(kMultiRows, hp.box[b].k - r0);
            th.push_back({hsrc * 16.0 * ((hr + 15) / 16) + 64.0, t});
          }
        }
      }
      std::stable_sort(th.begin(), th.end(),
                       [](const auto& x, const auto& y) { return x.first > y.first; });
      for (auto& e : th) hp.tasks_mh.push_back(e.second);
      // the u pass: longest first
      std::stable_sort(tv.begin(), tv.end(),
                       [](const auto& x, const auto& y) { return x.first > y.first; });
      for (auto& e : tv) hp.tasks_m.push_back(e.second);
      hp.n_tasks_mh = (int64_t)hp.tasks_mh.size();
    }

    // multi-RHS u pass with symmetric colleague blocks (single rank): the
    // block of an ifo pair b < c is generated once by b's tasks, which apply
    // it to b's rows (as kIFO) and, transposed, to b's charges for c's rows
    // (A_cb = A_bc^T): one staged n_c x kNRHS vector per (task, pair), added
    // by K2bm per receiving box in (b, task, entry) order -- deterministic.
    // The uhat pass keeps the unfolded lists (it visits ~1/8 of the columns).
    hp.multi_sym = hp.symmetric && n_ranks == 1 && opt.multi_sym;
    if (hp.multi_sym) {
      hp.ent_range_msym.resize(nb);
      std::vector<std::vector<int64_t>> inbox(nb);
      std::vector<std::pair<double, Task>> tv;
      int64_t cursor = 0;
      for (int32_t b = 0; b < nb; ++b) {
        EntryRange& er = hp.ent_range_msym[b];
        er.begin = (int64_t)hp.entries_msym.size();
        er.count = 0;
        if (d.box_level[b] < 1) continue;
        double cost = 0.0;
        int32_t soff = 0;
        sources(b, [&](int32_t c, int mode) {
          if (mode == kIFO && c != b) {
            if (c < b) return;  // arrives through b = c's staged column sums
            hp.entries_msym.push_back((c << kModeBits) | kSYM);
            hp.ent_soff_m.push_back(soff);
            soff += (hp.box[c].n + kChunkM - 1) / kChunkM * kChunkM;  // chunk-aligned (chain flags)
            cost += 1.6 * hp.box[c].n;  // one generation, two DMMA products
            return;
          }
          hp.entries_msym.push_back((c << kModeBits) | mode);
          hp.ent_soff_m.push_back(-1);
          cost += hp.box[c].n;
        });
        er.count = (int32_t)((int64_t)hp.entries_msym.size() - er.begin);
        if (er.count == 0) continue;
        // one staged vector per pair, shared by b's row tiles: tile t adds its
        // column sums to tile t-1's, chunk by chunk (chain flags), so the
        // staging is one n_c x kNRHS vector per pair, not per (pair, tile)
        int32_t tile = 0;
        for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += kMultiRows, ++tile)
          tv.push_back({cost * kMultiRows + 64.0,
                        Task{b, r0, std::min(kMultiRows, hp.box[b].n - r0), tile, cursor}});
        for (int64_t e = er.begin; e < er.begin + er.count; ++e)
          if (hp.ent_soff_m[e] >= 0)
            inbox[hp.entries_msym[e] >> kModeBits].push_back(cursor + hp.ent_soff_m[e]);
        cursor += soff;
      }
      hp.stage_m_points = cursor;
      // longest first; the tiles of a box keep their order (equal cost, stable
      // sort), so tile t - 1 is always claimed before tile t waits on it
      std::stable_sort(tv.begin(), tv.end(),
                       [](const auto& x, const auto& y) { return x.first > y.first; });
      hp.tasks_msym.reserve(tv.size());
      for (auto& e : tv) hp.tasks_msym.push_back(e.second);
      hp.recv_m_off.assign(1, 0);
      for (int32_t c = 0; c < nb; ++c) {
        if (inbox[c].empty()) continue;
        hp.recv_m_box.push_back(c);
        hp.recv_m_u.insert(hp.recv_m_u.end(), inbox[c].begin(), inbox[c].end());
        hp.recv_m_off.push_back((int64_t)hp.recv_m_u.size());
      }
    }

    ptime("multi csr");
    // ghost exchange lists: box c owned by p is sent to q if one of q's
    // targets reads it.  Every rank derives the same lists.
    if (n_ranks > 1) {
      std::vector<std::vector<uint8_t>> need(n_ranks, std::vector<uint8_t>(nb, 0));
      for (int32_t b = 0; b < nb; ++b) {
        if (d.box_level[b] < 1) continue;
        const int q = hp.owner[b];
        sources(b, [&](int32_t c, int mode) {
          if (hp.owner[c] == kShared) return;  // every rank holds shared boxes
          if (q == kShared) {                   // every rank evaluates b
            for (int p = 0; p < n_ranks; ++p)
              if (hp.owner[c] != p) need[p][c] = 1;
          } else if (hp.owner[c] != q && !folded_away(b, c, mode)) {
            need[q][c] = 1;
          }
        });
      }
      // shared boxes' slots that a child's upward pass fills (child owned by
      // p, parent shared): p sends them to every other rank
      std::vector<int32_t> shared_kids;
      if (hp.cut_level > 1)
        for (int32_t c = l1e; c < hp.level_begin[3]; ++c)
          if (hp.owner[d.box_parent[c]] == kShared && hp.box[c].k > 0) shared_kids.push_back(c);
      auto parent_slots = [&](int32_t c, std::vector<int64_t>& out) {
        const int64_t ps = hp.box[d.box_parent[c]].slot;
        for (int32_t i = 0; i < hp.box[c].k; ++i)
          out.push_back(ps + hp.posmap[ps + d.box_parent_offset[c] + i]);
      };
      auto parent_slots_global = [&](int32_t c, std::vector<int64_t>& out) {
        const int32_t pb = d.box_parent[c];
        const int64_t ps = hp.box[pb].slot, gs = hp.global_slot[pb];
        for (int32_t i = 0; i < hp.box[c].k; ++i)
          out.push_back(gs + hp.posmap[ps + d.box_parent_offset[c] + i]);
      };
      hp.send_off.assign(n_ranks + 1, 0);
      hp.recv_off_peer.assign(n_ranks + 1, 0);
      const int64_t sk_base = hp.n_slots;  // QH entries are addressed as n_slots + skel index
      // the same lists in the descriptor's (global) numbering, for the
      // host-only view (sfmm_gpu_shard_describe): they agree across ranks
      const bool compact = !hp.global_slot.empty();
      auto gslot = [&](int32_t c) { return compact ? hp.global_slot[c] : hp.box[c].slot; };
      auto gskel = [&](int32_t c) { return compact ? hp.global_skel[c] : hp.box[c].skel; };
      for (int p = 0; p < n_ranks; ++p) {
        for (int32_t c = 0; c < nb; ++c) {
          if (p != rank && need[p][c] && hp.owner[c] == rank) {  // I send c to p
            for (int32_t i = 0; i < hp.box[c].n; ++i) hp.pack_idx.push_back(hp.box[c].slot + i);
            for (int32_t i = 0; i < hp.box[c].k; ++i) hp.pack_idx.push_back(sk_base + hp.box[c].skel + i);
            if (compact) {
              for (int32_t i = 0; i < hp.box[c].n; ++i) hp.pack_idx_global.push_back(gslot(c) + i);
              for (int32_t i = 0; i < hp.box[c].k; ++i) hp.pack_idx_global.push_back(S + gskel(c) + i);
            }
          }
          if (p != rank && need[rank][c] && hp.owner[c] == p) {  // p sends c to me
            for (int32_t i = 0; i < hp.box[c].n; ++i) hp.unpack_idx.push_back(hp.box[c].slot + i);
            for (int32_t i = 0; i < hp.box[c].k; ++i) hp.unpack_idx.push_back(sk_base + hp.box[c].skel + i);
            if (compact) {
              for (int32_t i = 0; i < hp.box[c].n; ++i) hp.unpack_idx_global.push_back(gslot(c) + i);
              for (int32_t i = 0; i < hp.box[c].k; ++i) hp.unpack_idx_global.push_back(S + gskel(c) + i);
            }
            ++hp.n_ghost_boxes;
          }
        }
        for (int32_t c : shared_kids) {
          if (p != rank && hp.owner[c] == rank) {
            parent_slots(c, hp.pack_idx);
            if (compact) parent_slots_global(c, hp.pack_idx_global);
          }
          if (p != rank && hp.owner[c] == p) {
            parent_slots(c, hp.unpack_idx);
            if (compact) parent_slots_global(c, hp.unpack_idx_global);
          }
        }
        hp.send_off[p + 1] = (int64_t)hp.pack_idx.size();
        hp.recv_off_peer[p + 1] = (int64_t)hp.unpack_idx.size();
      }
    }

    ptime("ghost lists");
    // tasks: 128-row tiles of owned targets; staging slots for kSYM column
    // sums are assigned in (box, row tile, entry) order so every receiver adds
    // them in a fixed order.  Interior tasks (no ghost source) come first so
    // they can run while the ghost exchange is in flight.
    {
      std::vector<std::vector<std::pair<int64_t, int64_t>>> inbox(nb);
      std::vector<std::pair<double, Task>> tv_int, tv_bnd;
      int64_t cursor = 0;
      // cost model: lane-rows x (sources + 8)
      std::vector<double> src_of(nb, 0.0);
      for (int32_t b = 0; b < nb; ++b) {
        const EntryRange& er = hp.ent_range[b];
        for (int64_t e = er.begin; e < er.begin + er.count; ++e) {
          const int32_t code = hp.entries[e];
          const double w = (code & kModeMask) == kSYM ? 1.15 : 1.0;  // extra column accumulate
          src_of[b] += w * hp.box[code >> kModeBits].n;
        }
      }
      // Row-tile height: 128 (4 rows per lane) unless the tree is so small that
      // its largest tasks would set the persistent kernel's makespan (config-1
      // sized plans); then 64 or 32 rows.  Smaller tiles cost a little more
      // per pair (each staged source chunk serves fewer rows).
      int tile = kTileRows;
      {
        const double warps = 148.0 * 16.0;  // resident K2 warps on a B200
        double best = -1.0;
        for (int T : {kTileRows, kTileRows / 2, kTileRows / 4}) {
          double total = 0.0, longest = 0.0;
          for (int32_t b = 0; b < nb; ++b) {
            if (hp.ent_range[b].count == 0) continue;
            for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += T) {
              const int32_t rows = std::min(T, hp.box[b].n - r0);
              const double c = 32.0 * ((rows + 31) / 32) * (src_of[b] + 8.0);
              total += c;
              longest = std::max(longest, c);
            }
          }
          const double over = T == kTileRows ? 1.0 : (T == kTileRows / 2 ? 1.08 : 1.2);
          const double est = std::max(longest, over * total / warps);
          if (best < 0.0 || est < 0.9 * best) {  // a smaller tile must clearly win
            best = est;
            tile = T;
          }
        }
      }
#ifdef SFMM_TILE_FORCE
      tile = SFMM_TILE_FORCE;  // dev knob (A/B of the K2 occupancy variants)
#endif
      // rows per lane of the K2 instantiations this library was built with
      tile = std::min(tile, 32 * (hp.cplx ? SFMM_K2C_MAX_R : SFMM_K2_MAX_R));
      hp.tile_rows = tile;
      // Source-range split (single-rank real plans of 32-row tiles, small enough
      // for one task to set the persistent kernel's makespan, config 1): a row tile
      // costing more than 3/4 of the per-warp share of the work is cut along
      // its entry list into parts of about half a share.  The first part owns
      // the rows as usual; each later part leaves raw row partials in a
      // zero-filled [u: n_b | h: k_b] staging vector (rows outside the tile are
      // never written) that K2b adds to the box in the fixed part order.
      double split_share = 0.0;
      if (n_ranks == 1 && !hp.cplx && !hp.sym_chain && opt.split && !opt.merge_tiles &&
          tile <= 32) {
        double total = 0.0;
        for (int32_t b = 0; b < nb; ++b) {
          if (hp.ent_range[b].count == 0) continue;
          for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += tile)
            total += 32.0 * ((std::min(tile, hp.box[b].n - r0) + 31) / 32) * (src_of[b] + 8.0);
        }
        split_share = total / (148.0 * 32.0);  // resident warps of the 32-row (R = 1) K2
      }
      // Merged tasks: a box of several row tiles whose whole cost stays well
      // below the per-warp share is ONE task; the kernel runs its tiles in
      // order and every tile continues the kSYM column sums of one staged
      // vector per pair (the chained layout's memory, without the chain's
      // cross-warp waits).
      double merge_cap = 0.0;
      if (opt.merge_tiles && !hp.sym_chain && split_share == 0.0) {
        double total = 0.0;
        for (int32_t b = 0; b < nb; ++b) {
          if (hp.ent_range[b].count == 0) continue;
          for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += tile)
            total += 32.0 * ((std::min(tile, hp.box[b].n - r0) + 31) / 32) * (src_of[b] + 8.0);
        }
        merge_cap = opt.merge_share * total / (148.0 * 16.0);
      }
      // outgoing cross-rank pairs in (b, entry) order, the staged tiles of each
      std::vector<std::pair<int32_t, int32_t>> xpairs;
      std::vector<std::vector<std::pair<int64_t, int64_t>>> xtiles;
      for (int32_t b = 0; b < nb; ++b) {
        const EntryRange& er = hp.ent_range[b];
        const size_t x0 = xpairs.size();
        for (int64_t e = er.begin; e < er.begin + er.count; ++e) {
          const int32_t code = hp.entries[e];
          if ((code & kModeMask) == kSYM && !mine(code >> kModeBits))
            xpairs.push_back({b, code >> kModeBits});
        }
        xtiles.resize(xpairs.size());
        if (er.count == 0 || hp.box[b].n == 0) continue;
        const double src = src_of[b];
        // Staged [u: n_c | h: k_c] vectors of the kSYM pairs (b, c), each on a
        // 32-scalar boundary (chain flags are offset / 32 + column / 32):
        // one per (pair, row tile) -- the tile owning skeleton rows carries
        // the h part -- or, with sym_chain, one per pair shared by all of b's
        // row tiles, tile t adding to tile t - 1's in tile order.
        auto stage_entries = [&](bool h_part, int64_t e_from = 0, int64_t e_to = -1) {
          size_t xi = x0;  // (parts: single-rank plans only, so no cross-rank pairs)
          for (int64_t e = er.begin + e_from; e < er.begin + (e_to < 0 ? er.count : e_to); ++e) {
            const int32_t code = hp.entries[e];
            if ((code & kModeMask) != kSYM) continue;
            const int32_t c = code >> kModeBits;
            const int64_t u_off = cursor;
            int64_t h_off = -1;
            int64_t len = hp.box[c].n;
            if (h_part && hp.box[c].k > 0) {
              h_off = cursor + hp.box[c].n;
              len += hp.box[c].k;
            }
            cursor += (len + 31) & ~(int64_t)31;
            if (mine(c))
              inbox[c].push_back({u_off, h_off});
            else
              xtiles[xi++].push_back({u_off, h_off});
          }
        };
        const int64_t b_stage = cursor;
        if (merge_cap > 0.0 && hp.box[b].n > tile) {
          double cost = 0.0;
          for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += tile)
            cost += 32.0 * ((std::min(tile, hp.box[b].n - r0) + 31) / 32) * (src + 8.0);
          if (cost <= merge_cap) {
            stage_entries(hp.box[b].k > 0);
            auto& tv = (boundary[b] || !opt.overlap) ? tv_bnd : tv_int;
            tv.push_back({cost, Task{b, 0, hp.box[b].n, -1, b_stage}});
            ++hp.n_merged_tasks;
            continue;
          }
        }
        if (hp.sym_chain) stage_entries(hp.box[b].k > 0);
        int32_t tile_index = 0;
        for (int32_t r0 = 0; r0 < hp.box[b].n; r0 += tile, ++tile_index) {
          Task t{b, r0, std::min(tile, hp.box[b].n - r0), hp.sym_chain ? tile_index : -1,
                 hp.sym_chain ? b_stage : cursor};
          const double lanes_rows = 32.0 * ((t.nrows + 31) / 32);
          const double cost = lanes_rows * (src + 8.0);
          // without overlap every task runs in the one launch after the exchange
          auto& tv = (boundary[b] || !opt.overlap) ? tv_bnd : tv_int;
          if (split_share > 0.0 && cost > 1.5 * opt.split_part * split_share && er.count > 1) {
            const bool skel = r0 < hp.box[b].k;
            int32_t e0 = 0;
            double acc = 0.0;
            for (int32_t e = 0; e < er.count; ++e) {
              const int32_t code = hp.entries[er.begin + e];
              acc += lanes_rows * ((code & kModeMask) == kSYM ? 1.15 : 1.0) * hp.box[code >> kModeBits].n;
              if (acc < opt.split_part * split_share && e + 1 < er.count) continue;
              Task part = t;
              part.stage = cursor;
              part.e0 = e0;
              part.e1 = e + 1;
              stage_entries(skel, e0, e + 1);
              if (e0 > 0) {  // a later part: its row-partial vector
                part.rstage = cursor;
                inbox[b].push_back({cursor, skel ? cursor + hp.box[b].n : -1});
                cursor += (hp.box[b].n + (skel ? hp.box[b].k : 0) + 31) & ~(int64_t)31;
                ++hp.n_split_parts;
              }
              tv.push_back({acc + lanes_rows * 8.0, part});
              e0 = e + 1;
              acc = 0.0;
            }
            continue;
          }
          if (!hp.sym_chain) stage_entries(r0 < hp.box[b].k);
          tv.push_back({cost, t});
        }
      }
      hp.stage_size = cursor;
      // Second exchange: one vector per (peer, receiving box c) -- the column
      // sums of every pair (b, c) this rank evaluated, summed over b and b's
      // row tiles by k_xpack -- in ascending c per peer.  The receiver rebuilds
      // the list from the global tree.  The h part exists iff some pair of the
      // group has skeletons on both sides.
      if (hp.xsym) {
        auto has_h = [&](int32_t b, int32_t c) { return hp.box[b].k > 0 && hp.box[c].k > 0; };
        std::vector<int32_t> ord(xpairs.size());
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
          const int32_t cx = xpairs[x].second, cy = xpairs[y].second;
          if (hp.owner[cx] != hp.owner[cy]) return hp.owner[cx] < hp.owner[cy];
          return cx < cy;
        });
        hp.send2_off.assign(n_ranks + 1, 0);
        hp.recv2_off.assign(n_ranks + 1, 0);
        hp.xpair_tile_off.assign(1, 0);
        int64_t dst = 0;
        for (size_t g = 0; g < ord.size();) {
          const int32_t c = xpairs[ord[g]].second;
          bool h = false;
          for (; g < ord.size() && xpairs[ord[g]].second == c; ++g) {
            h = h || has_h(xpairs[ord[g]].first, c);
            for (auto& uh : xtiles[ord[g]]) {
              hp.xtile_u.push_back(uh.first);
              hp.xtile_h.push_back(uh.second);
            }
          }
          const int32_t nh = h ? hp.box[c].k : 0;
          hp.xpair_tile_off.push_back((int64_t)hp.xtile_u.size());
          hp.xpair_dst.push_back(dst);
          hp.xpair_nu.push_back(hp.box[c].n);
          hp.xpair_nh.push_back(nh);
          dst += hp.box[c].n + nh;
          hp.send2_off[hp.owner[c] + 1] = dst;
        }
        for (int p = 0; p < n_ranks; ++p)
          hp.send2_off[p + 1] = std::max(hp.send2_off[p + 1], hp.send2_off[p]);
        int64_t src2 = 0;
        for (int p = 0; p < n_ranks; ++p) {
          if (p != rank)
            for (int32_t c = hp.level_begin[2]; c < nb; ++c) {
              if (!mine(c)) continue;
              bool any = false, h = false;
              for (int64_t e = d.coll_off[c]; e < d.coll_off[c + 1]; ++e) {
                const int32_t b = d.coll[e];
                if (hp.owner[b] != p || (unc[b] && unc[c]) || !evaluates(b, c)) continue;
                any = true;
                h = h || has_h(b, c);
              }
              if (!any) continue;
              const int64_t u_off = hp.stage_size + src2;
              src2 += hp.box[c].n;
              int64_t h_off = -1;
              if (h) {
                h_off = hp.stage_size + src2;
                src2 += hp.box[c].k;
              }
              inbox[c].push_back({u_off, h_off});
            }
          hp.recv2_off[p + 1] = src2;
        }
      }
#ifndef SFMM_TASK_GROUP_R
#define SFMM_TASK_GROUP_R 1
#endif
      // Longest first (LPT) by cost band (factor 1.25), and by rows-per-lane R
      // (the K2 code path) within a band, so the warps resident together
      // mostly run one instantiation -- mixing all four R variants starves
      // instruction fetch on adaptive trees -- without pushing expensive
      // partial tiles to the tail.
      auto band = [](double c) { return (int)std::floor(std::log(c + 1.0) / std::log(1.25)); };
      auto by_cost = [&](const auto& a, const auto& b) {
        if (SFMM_TASK_GROUP_R) {
          const int ba = band(a.first), bb = band(b.first);
          if (ba != bb) return ba > bb;
          const int ra = (a.second.nrows + 31) >> 5, rb = (b.second.nrows + 31) >> 5;
          if (ra != rb) return ra > rb;
        }
        return a.first > b.first;
      };
      std::stable_sort(tv_int.begin(), tv_int.end(), by_cost);
      std::stable_sort(tv_bnd.begin(), tv_bnd.end(), by_cost);
      hp.tasks.reserve(tv_int.size() + tv_bnd.size());
      for (auto& e : tv_int) hp.tasks.push_back(e.second);
      hp.n_interior_tasks = (int64_t)tv_int.size();
      for (auto& e : tv_bnd) hp.tasks.push_back(e.second);
      hp.recv_off.assign(1, 0);
      for (int32_t c = 0; c < (int32_t)inbox.size(); ++c) {
        if (inbox[c].empty()) continue;
        hp.recv_box.push_back(c);
        for (auto& uh : inbox[c]) {
          hp.recv_u.push_back(uh.first);
          hp.recv_h.push_back(uh.second);
        }
        hp.recv_off.push_back((int64_t)hp.recv_u.size());
      }
    }

    ptime("tasks");
    // interpolation work lists per level (owned boxes at levels >= 2 carry T);
    // T is compacted to the owned boxes (T_off indexes the compact blob)
    hp.T_off.assign(nb + 1, 0);
    hp.T_runs.clear();
    int64_t tcur = 0;
    for (int32_t b = 0; b < nb; ++b) {
      hp.T_off[b] = tcur;
      const int64_t len = d.T_off[b + 1] - d.T_off[b];
      if (len > 0 && mine(b)) {
        if (!hp.T_runs.empty() && hp.T_runs.back().src + hp.T_runs.back().len == d.T_off[b] &&
            hp.T_runs.back().dst + hp.T_runs.back().len == tcur)
          hp.T_runs.back().len += len;
        else
          hp.T_runs.push_back({d.T_off[b], tcur, len});
        tcur += len;
      }
    }
    hp.T_off[nb] = tcur;
    hp.up_lvl.assign(d.depth + 2, 0);
    hp.up1_lvl.assign(d.depth + 2, 0);
    hp.copy_lvl.assign(d.depth + 2, 0);
    hp.copy_dn_lvl.assign(d.depth + 2, 0);
    hp.down_lvl.assign(d.depth + 2, 0);
    hp.down_m_lvl.assign(d.depth + 2, 0);
    for (int l = 0; l <= d.depth; ++l) {
      hp.up_lvl[l] = (int64_t)hp.up_items.size();
      hp.up1_lvl[l] = (int64_t)hp.up1_items.size();
      hp.copy_lvl[l] = (int64_t)hp.copy_boxes.size();
      hp.copy_dn_lvl[l] = (int64_t)hp.copy_boxes_dn.size();
      hp.down_lvl[l] = (int64_t)hp.down_items.size();
      hp.down_m_lvl[l] = (int64_t)hp.down_m_items.size();
      if (l >= 2) {
        for (int32_t b = hp.level_begin[l]; b < hp.level_begin[l + 1]; ++b) {
          if (!mine(b)) continue;
          const int32_t k = hp.box[b].k, r = hp.box[b].n - hp.box[b].k;
          if (k == 0) continue;
          for (int32_t i = 0; i < k; i += kUpRows) hp.up_items.push_back({b, i});
          // one K3m item even when r == 0: it also folds uhat into the skeleton slots
          for (int32_t j = 0; j < std::max(r, 1); j += kDownColsM) hp.down_m_items.push_back({b, j});
          if (r == 0) {  // uncompressed: copies only (warp per box, k1_copy / k3_copy;
                         // leaves: fused into K0 / K4)
            if (!d.box_leaf[b]) {
              hp.copy_boxes.push_back(b);
              hp.copy_boxes_dn.push_back(b);
            }
            continue;
          }
          if (r <= kWarpBoxR) {  // short interpolation block: warp per box upward
            hp.copy_boxes.push_back(b);
            for (int32_t j = 0; j < r; j += kDownCols) hp.down_items.push_back({b, j});
            continue;
          }
          for (int32_t i = 0; i < k; i += kUpRows1) hp.up1_items.push_back({b, i});
          for (int32_t j = 0; j < r; j += kDownCols) hp.down_items.push_back({b, j});
        }
      }
    }
    ptime("T runs, level items");
    hp.up_lvl[d.depth + 1] = (int64_t)hp.up_items.size();
    hp.up1_lvl[d.depth + 1] = (int64_t)hp.up1_items.size();
    hp.copy_lvl[d.depth + 1] = (int64_t)hp.copy_boxes.size();
    hp.copy_dn_lvl[d.depth + 1] = (int64_t)hp.copy_boxes_dn.size();
    hp.down_lvl[d.depth + 1] = (int64_t)hp.down_items.size();
    hp.down_m_lvl[d.depth + 1] = (int64_t)hp.down_m_items.size();
    // persistent tree passes (opt-in A/B, plan_build.h kTreePersistPoints)
    {
      hp.tree_persist = opt.tree_persist >= 0 ? opt.tree_persist != 0
                                              : (hp.n_owned_points > 0 && hp.n_owned_points <= kTreePersistPoints);
      if (hp.tree_persist) {
        const int32_t n_pj = (int32_t)((hp.n_owned_points + kPointsPerJob - 1) / kPointsPerJob);
        auto level_jobs = [&](int l, const std::vector<int64_t>& lvl, std::vector<TreeJob>& jobs,
                              int32_t stage) {
          const std::vector<int64_t>& cl = &lvl == &hp.up1_lvl ? hp.copy_lvl : hp.copy_dn_lvl;
          for (int64_t c = cl[l]; c < cl[l + 1]; c += 8)
            jobs.push_back({kJobCopy, stage, (int32_t)c, (int32_t)std::min<int64_t>(8, cl[l + 1] - c)});
          for (int64_t i = lvl[l]; i < lvl[l + 1]; ++i) jobs.push_back({kJobItem, stage, (int32_t)i, 0});
        };
        int32_t stage = 0;
        for (int32_t j = 0; j < n_pj; ++j) hp.up_jobs.push_back({kJobGather, 0, j, 0});
        for (int l = d.depth; l >= 2; --l) level_jobs(l, hp.up1_lvl, hp.up_jobs, ++stage);
        auto firsts = [](const std::vector<TreeJob>& jobs, int32_t n_stages) {
          std::vector<int32_t> f(n_stages + 1, 0);
          for (const TreeJob& j : jobs) ++f[j.stage + 1];
          for (int32_t i = 0; i < n_stages; ++i) f[i + 1] += f[i];
          return f;
        };
        hp.up_stage_first = firsts(hp.up_jobs, stage + 1);
        stage = 0;
        for (int l = 2; l <= d.depth; ++l, ++stage)
          level_jobs(l, hp.down_lvl, hp.down_jobs, stage);
        for (int32_t j = 0; j < n_pj; ++j) hp.down_jobs.push_back({kJobScatter, stage, j, 0});
        hp.down_stage_first = firsts(hp.down_jobs, stage + 1);
      }
    }
    return SFMM_OK;
  } catch (const Fail& f) {
    err = f.msg;
    return f.code;
  } catch (const std::bad_alloc&) {
    err = "sfmm_gpu_plan_create: host allocation failed";
    return SFMM_ENOMEM;
  }
}

}  // namespace sfmm_gpu
