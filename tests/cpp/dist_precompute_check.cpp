// C++ check of the distributed precompute (include/sfmm_gpu_dist.hpp) on one
// GPU: R virtual ranks each build the tree, skeletonize their own subtrees and
// contribute their index data; the descriptor every rank assembles and every
// rank's operators must equal the whole-tree build exactly, and every rank
// plan must build (sfmm_gpu_plan_create_sharded_owned).
//   dist_precompute_check <n_ranks> <n_points> <kernel: 1 Laplace3d, 3 Helmholtz3d>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <vector>

#include "sfmm_gpu_dist.hpp"

namespace {

template <class T>
bool same(const char* what, const T* a, const T* b, int64_t n) {
  if (n == 0 || std::memcmp(a, b, sizeof(T) * n) == 0) return true;
  std::fprintf(stderr, "mismatch: %s\n", what);
  return false;
}

}  // namespace

int main(int argc, char** argv) {
  const int n_ranks = argc > 1 ? std::atoi(argv[1]) : 4;
  const int64_t n = argc > 2 ? std::atoll(argv[2]) : 60000;
  const int kernel = argc > 3 ? std::atoi(argv[3]) : SFMM_LAPLACE3D;
  const double kappa = kernel == SFMM_HELMHOLTZ3D ? 10.0 : 0.0;
  const int sw = kernel == SFMM_HELMHOLTZ3D ? 2 : 1;
  std::mt19937_64 rng(7);
  std::vector<double> pts(3 * n);
  for (double& x : pts) x = (rng() >> 11) * 0x1.0p-53;
  try {
    // the whole-tree build
    sfmm_gpu_tree* tree = nullptr;
    sfmm_tree_arrays ta{};
    if (sfmm_gpu_build_tree(3, n, pts.data(), 64, 0, &tree) || sfmm_gpu_tree_arrays(tree, &ta))
      throw std::runtime_error(sfmm_gpu_last_error());
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
    sfmm_skel_result* full = nullptr;
    sfmm_plan_desc fd{};
    if (sfmm_gpu_build_skeletons(&td, kernel, kappa, 1e-6, 0.0, 0, 0, 0, &full) ||
        sfmm_gpu_skel_describe(full, &fd, 1, nullptr, nullptr, nullptr, nullptr))
      throw std::runtime_error(sfmm_gpu_last_error());
    const int32_t nb = ta.n_boxes;
    // the ranks
    std::vector<std::unique_ptr<sfmm::gpu::RankPrecompute>> pre;
    std::vector<sfmm::gpu::IndexPart> parts;
    for (int r = 0; r < n_ranks; ++r) {
      pre.emplace_back(new sfmm::gpu::RankPrecompute(kernel, kappa, 3, n, pts.data(), 64, 1e-6,
                                                     n_ranks, r, 0));
      parts.push_back(pre.back()->part());
    }
    bool ok = true;
    for (int r = 0; r < n_ranks && ok; ++r) {
      const sfmm_plan_desc& d = pre[r]->assemble(parts);
      ok = same("iv_off", d.iv_off, fd.iv_off, nb + 1) && same("sk_off", d.sk_off, fd.sk_off, nb + 1) &&
           same("rd_off", d.rd_off, fd.rd_off, nb + 1) && same("T_off", d.T_off, fd.T_off, nb + 1) &&
           same("iv", d.iv, fd.iv, fd.iv_off[nb]) && same("skel_pos", d.skel_pos, fd.skel_pos, fd.sk_off[nb]) &&
           same("red_pos", d.red_pos, fd.red_pos, fd.rd_off[nb]) &&
           same("parent_offset", d.box_parent_offset, fd.box_parent_offset, nb);
      // the rank's operators = the full T of its boxes, in box order
      int64_t nt = 0;
      const double* T = pre[r]->host_T(&nt);
      int64_t at = 0;
      const std::vector<int32_t>& own = pre[r]->owner();
      for (int32_t b = 0; b < nb && ok; ++b) {
        if (own[b] != r) continue;
        const int64_t len = (fd.T_off[b + 1] - fd.T_off[b]) * sw;
        ok = at + len <= nt && same("T", T + at, fd.T + fd.T_off[b] * sw, len);
        at += len;
      }
      ok = ok && at == nt;
    }
    for (int r = 0; r < n_ranks && ok; ++r) {
      sfmm_gpu_plan* p = pre[r]->make_plan(parts);
      sfmm_gpu_plan_destroy(p);
    }
    sfmm_gpu_skel_destroy(full);
    sfmm_gpu_tree_destroy(tree);
    std::printf("%s: %d ranks, %lld points, %d boxes\n", ok ? "ok" : "FAILED", n_ranks, (long long)n, nb);
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
