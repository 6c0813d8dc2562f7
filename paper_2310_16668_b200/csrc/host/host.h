// Host copies of a plan built on the GPU (tree, neighbor lists, skeletons).
#pragma once

#include <stdint.h>

#include <array>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfmm_host {

struct Box {
  int32_t parent = -1;
  int32_t child[8] = {-1, -1, -1, -1, -1, -1, -1, -1};  // by octant
  int32_t level = 0;
  uint64_t morton = 0;
  int64_t cell[3] = {0, 0, 0};
  double center[3] = {0, 0, 0};
  double half = 0;
  int32_t begin = 0, end = 0;
  bool leaf = false;
  int32_t npoints() const { return end - begin; }
};

// Level-major, Morton-sorted tree (same layout as sfmm::Tree, tree.hpp:19-52).
struct Tree {
  int dim = 0, depth = 0, leaf_cap = 0;
  std::vector<Box> boxes;
  std::vector<int32_t> level_begin;  // depth + 2
  std::vector<int32_t> perm;         // tree position -> original index
  std::vector<double> pts;           // tree order, interleaved
};

struct Neighbors {
  // CSR per box
  std::vector<int64_t> coll_off, coarse_off, fine_off;
  std::vector<int32_t> coll, coarse, fine;
};

// Skeleton data in CSR form (the sfmm_plan_desc layout).
struct Skeletons {
  std::vector<int64_t> iv_off, sk_off, rd_off, T_off;
  std::vector<int32_t> iv, skel_pos, red_pos, parent_offset;
  std::vector<double> T;  // complex: interleaved
  int k_max = 0;
  int saturated = 0;
  int64_t proj_scalars = 0;
};

// Synthetic inputs (bench.cpp:25-45,102-161 definitions).
void generate_points(int dist, int64_t n, uint64_t seed, double* out);
void generate_charges(int64_t n, uint64_t seed, double* out);
void generate_charges_complex(int64_t n, uint64_t seed, double* out);

}  // namespace sfmm_host
