// sfmm_gpu_dist.hpp -- header-only C++ for the distributed precompute of a
// sharded plan (config 5 scale: no rank ever holds every operator).
//
// One process per GPU.  Every rank builds the same tree on its GPU, takes the
// tree-only ownership of the level-1 subtrees, skeletonizes only its own
// subtrees (operators stay in its HBM), contributes the index data of its
// boxes (a few bytes per point) to an all-gather of the caller's transport
// (MPI_Allgatherv, NCCL, files), and builds its rank plan from the assembled
// descriptor and its own operators:
//
//     sfmm::gpu::RankPrecompute pre(SFMM_LAPLACE3D, 0.0, 3, n, pts, 128, 1e-6,
//                                   n_ranks, rank, local_gpu);
//     std::vector<sfmm::gpu::IndexPart> all = my_allgather(pre.part());
//     sfmm_gpu_plan* plan = pre.make_plan(all);       // then attach NCCL, apply
//
// Needs only sfmm_gpu.h (no reference headers); shard.distributed_precompute is
// the same flow in Python.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfmm_gpu.h"

namespace sfmm {
namespace gpu {

// One rank's share of the skeleton index data: for each box it owns (ascending
// id) its index_vec / skel_pos / red_pos segment lengths and contents and its
// parent_offset.
struct IndexPart {
  std::vector<int32_t> boxes, poff;
  std::vector<int64_t> len_iv, len_sk, len_rd;
  std::vector<int32_t> iv, sk, rd;
};

class RankPrecompute {
 public:
  RankPrecompute(int kernel, double kappa, int dim, int64_t n, const double* pts, int leaf_cap,
                 double tol, int n_ranks, int rank, int device)
      : kernel_(kernel), kappa_(kappa), n_ranks_(n_ranks), rank_(rank), device_(device) {
    check(sfmm_gpu_build_tree(dim, n, pts, leaf_cap, device, &tree_), "build_tree");
    check(sfmm_gpu_tree_arrays(tree_, &ta_), "tree_arrays");
    owner_.resize(ta_.n_boxes);
    check(sfmm_gpu_subtree_owners(&ta_, n_ranks, owner_.data()), "subtree_owners");
    std::vector<uint8_t> mine(ta_.n_boxes);
    for (int32_t b = 0; b < ta_.n_boxes; ++b) mine[b] = owner_[b] == rank ? 1 : 0;
    sfmm_tree_desc td{};
    td.dim = ta_.dim;
    td.n_points = ta_.n_points;
    td.n_boxes = ta_.n_boxes;
    td.depth = ta_.depth;
    td.pts = ta_.pts;
    td.level_begin = ta_.level_begin;
    td.box_parent = ta_.box_parent;
    td.box_level = ta_.box_level;
    td.box_begin = ta_.box_begin;
    td.box_end = ta_.box_end;
    td.box_leaf = ta_.box_leaf;
    td.box_center = ta_.box_center;
    td.box_half = ta_.box_half;
    check(sfmm_gpu_build_skeletons_subset(&td, kernel, kappa, tol, 0.0, 0, 0, device, mine.data(),
                                          &skel_),
          "build_skeletons_subset");
    sfmm_plan_desc loc{};
    check(sfmm_gpu_skel_describe(skel_, &loc, 0, nullptr, nullptr, nullptr, nullptr), "skel_describe");
    // the subset result leaves every other box empty: its packed arrays are
    // exactly the owned boxes' segments in box order
    const int32_t nb = ta_.n_boxes;
    for (int32_t b = 0; b < nb; ++b) {
      if (owner_[b] != rank) continue;
      part_.boxes.push_back(b);
      part_.poff.push_back(loc.box_parent_offset[b]);
      part_.len_iv.push_back(loc.iv_off[b + 1] - loc.iv_off[b]);
      part_.len_sk.push_back(loc.sk_off[b + 1] - loc.sk_off[b]);
      part_.len_rd.push_back(loc.rd_off[b + 1] - loc.rd_off[b]);
    }
    part_.iv.assign(loc.iv, loc.iv + loc.iv_off[nb]);
    part_.sk.assign(loc.skel_pos, loc.skel_pos + loc.sk_off[nb]);
    part_.rd.assign(loc.red_pos, loc.red_pos + loc.rd_off[nb]);
  }

  RankPrecompute(const RankPrecompute&) = delete;
  RankPrecompute& operator=(const RankPrecompute&) = delete;
  ~RankPrecompute() {
    if (skel_) sfmm_gpu_skel_destroy(skel_);
    if (tree_) sfmm_gpu_tree_destroy(tree_);
  }

  const IndexPart& part() const { return part_; }
  const std::vector<int32_t>& owner() const { return owner_; }

  // The full descriptor (no T) from every rank's part, in rank order; its
  // arrays live in this object.
  const sfmm_plan_desc& assemble(const std::vector<IndexPart>& all) {
    const int32_t nb = ta_.n_boxes;
    std::vector<int64_t> liv(nb, 0), lsk(nb, 0), lrd(nb, 0);
    poff_.assign(nb, 0);
    for (const IndexPart& p : all)
      for (size_t i = 0; i < p.boxes.size(); ++i) {
        const int32_t b = p.boxes[i];
        liv[b] = p.len_iv[i];
        lsk[b] = p.len_sk[i];
        lrd[b] = p.len_rd[i];
        poff_[b] = p.poff[i];
      }
    auto offsets = [nb](const std::vector<int64_t>& len, std::vector<int64_t>& off) {
      off.assign(nb + 1, 0);
      for (int32_t b = 0; b < nb; ++b) off[b + 1] = off[b] + len[b];
    };
    offsets(liv, iv_off_);
    offsets(lsk, sk_off_);
    offsets(lrd, rd_off_);
    auto place = [](const IndexPart& p, const std::vector<int64_t>& part_len,
                    const std::vector<int32_t>& src, const std::vector<int64_t>& off,
                    std::vector<int32_t>& dst) {
      int64_t s = 0;
      for (size_t i = 0; i < p.boxes.size(); ++i) {
        for (int64_t e = 0; e < part_len[i]; ++e) dst[off[p.boxes[i]] + e] = src[s + e];
        s += part_len[i];
      }
    };
    iv_.assign(iv_off_[nb], 0);
    sk_.assign(sk_off_[nb], 0);
    rd_.assign(rd_off_[nb], 0);
    for (const IndexPart& p : all) {
      place(p, p.len_iv, p.iv, iv_off_, iv_);
      place(p, p.len_sk, p.sk, sk_off_, sk_);
      place(p, p.len_rd, p.rd, rd_off_, rd_);
    }
    T_off_.assign(nb + 1, 0);
    for (int32_t b = 0; b < nb; ++b)
      T_off_[b + 1] = T_off_[b] + (ta_.box_level[b] >= 2 ? lsk[b] * (liv[b] - lsk[b]) : 0);
    sfmm_plan_desc& d = desc_;
    d = sfmm_plan_desc{};
    d.kernel = kernel_;
    d.dim = ta_.dim;
    d.kappa = kappa_;
    d.n_points = ta_.n_points;
    d.n_boxes = nb;
    d.depth = ta_.depth;
    d.pts = ta_.pts;
    d.perm = ta_.perm;
    d.level_begin = ta_.level_begin;
    d.box_parent = ta_.box_parent;
    d.box_level = ta_.box_level;
    d.box_begin = ta_.box_begin;
    d.box_end = ta_.box_end;
    d.box_leaf = ta_.box_leaf;
    d.box_parent_offset = poff_.data();
    d.iv_off = iv_off_.data();
    d.iv = iv_.data();
    d.sk_off = sk_off_.data();
    d.skel_pos = sk_.data();
    d.rd_off = rd_off_.data();
    d.red_pos = rd_.data();
    d.T_off = T_off_.data();
    d.T = nullptr;
    d.coll_off = ta_.coll_off;
    d.coll = ta_.coll;
    d.coarse_off = ta_.coarse_off;
    d.coarse = ta_.coarse;
    d.fine_off = ta_.fine_off;
    d.fine = ta_.fine;
    return d;
  }

  // This rank's plan from the assembled descriptor and its own operators
  // (sfmm_gpu_plan_create_sharded_owned); the caller owns the plan.
  sfmm_gpu_plan* make_plan(const std::vector<IndexPart>& all) {
    const sfmm_plan_desc& d = assemble(all);
    const double* T = sfmm_gpu_skel_device_T(skel_, nullptr, nullptr);
    sfmm_gpu_plan* p = nullptr;
    check(sfmm_gpu_plan_create_sharded_owned(&d, T, device_, n_ranks_, rank_, owner_.data(), &p),
          "plan_create_sharded_owned");
    return p;
  }

  // This rank's operators (its subtrees' T in box order): on the device, or a
  // host copy (downloaded once, held by the skeleton result).
  const double* device_T(int64_t* n_scalars) const {
    return sfmm_gpu_skel_device_T(skel_, nullptr, n_scalars);
  }
  const double* host_T(int64_t* n_scalars) {
    sfmm_plan_desc tmp{};
    check(sfmm_gpu_skel_describe(skel_, &tmp, 1, nullptr, nullptr, nullptr, nullptr), "skel_describe");
    sfmm_gpu_skel_device_T(skel_, nullptr, n_scalars);
    return tmp.T;
  }

 private:
  static void check(int rc, const char* what) {
    if (rc != SFMM_OK)
      throw std::runtime_error(std::string("RankPrecompute: ") + what + ": " + sfmm_gpu_last_error());
  }

  int kernel_;
  double kappa_;
  int n_ranks_, rank_, device_;
  sfmm_gpu_tree* tree_ = nullptr;
  sfmm_tree_arrays ta_{};
  sfmm_skel_result* skel_ = nullptr;
  std::vector<int32_t> owner_;
  IndexPart part_;
  sfmm_plan_desc desc_{};
  std::vector<int64_t> iv_off_, sk_off_, rd_off_, T_off_;
  std::vector<int32_t> iv_, sk_, rd_, poff_;
};

}  // namespace gpu
}  // namespace sfmm
