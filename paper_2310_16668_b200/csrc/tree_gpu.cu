// GPU tree and neighbor lists.
//
// Device counterpart of build_tree + build_neighbors
// (/root/reference/proj/src/tree.cpp:148-355), bit-identical to the reference:
// same perm, level-major Morton box order, point ranges and lists (pinned by
// tests/test_tree_gpu.py against the reference and the host builder).
//
//   refine      level-synchronous on the device.  At each level the points of
//               the boxes above the leaf capacity are compacted and stably
//               radix-sorted by (box rank, octant) -- exactly the reference's
//               stable per-box partition -- and the non-empty children are
//               created in octant order with the reference's centre / half
//               arithmetic, so every level comes out Morton-sorted.
//   duplicates  coincident points always share a leaf, so a leaf-local
//               pairwise check replaces the reference's global sort
//               (tree.cpp:160); the host sort runs only to word the error (and
//               before reporting an unreachable leaf capacity, as the
//               reference checks duplicates first).
//   balance     the reference replays a (level, Morton)-ordered work queue and
//               the set of forced splits depends on that order (empty
//               children are pruned).  A leaf that satisfies 2:1 after
//               refinement can never violate it later (splits only deepen the
//               covering boxes, and a non-leaf cover never grows its missing
//               child), so the device flags the violating leaves in parallel
//               and only they seed the sequential replay on the host, which
//               is then equivalent to the reference's full queue.
//   neighbors   colleague / coarse / fine lists by binary search in the
//               level-sorted Morton codes, one thread per box.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "sfmm_gpu.h"

namespace sfmm_gpu {
int set_last_error(int code, const std::string& msg);
}

struct sfmm_gpu_tree {
  int dim = 0, depth = 0, leaf_cap = 0;
  int64_t n = 0;
  std::vector<int32_t> perm, level_begin, parent, child, level, begin, end;
  std::vector<double> pts, center, half;
  std::vector<uint64_t> morton;
  std::vector<int64_t> cell;
  std::vector<uint8_t> leaf;
  std::vector<int64_t> coll_off, coarse_off, fine_off;
  std::vector<int32_t> coll, coarse, fine;
  double seconds = 0;
};

namespace {

constexpr int kMaxDepth2 = 31, kMaxDepth3 = 21;  // 64-bit Morton budget (tree.hpp:15)
constexpr int kDupLeafMax = 2048;                 // larger leaves: host duplicate sort

struct TreeFail {
  int code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  (void)cudaGetLastError();  // reported here; do not leak into the next call
  throw TreeFail{e == cudaErrorMemoryAllocation ? SFMM_ENOMEM : SFMM_ECUDA,
                 std::string("build_tree: ") + what + ": " + cudaGetErrorString(e)};
}

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

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t c) { alloc(c); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  void alloc(size_t c) {
    if (p) cudaFree(p);
    p = nullptr;
    n = c;
    ck(cudaMalloc(&p, std::max<size_t>(c, 1) * sizeof(T)), "cudaMalloc");
  }
  void grow(size_t c) {
    if (c > n || !p) alloc(c);
  }
  void upload(const T* src, size_t c) {
    alloc(c);
    if (c) ck(cudaMemcpy(p, src, c * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  void download(T* dst, size_t c) const {
    if (c) ck(cudaMemcpy(dst, p, c * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }
  T get(size_t i) const {
    T v;
    ck(cudaMemcpy(&v, p + i, sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    return v;
  }
};

// One box of a level during construction.
struct LBox {
  double c[3];
  double half;
  uint64_t morton;
  int32_t cell[3];
  int32_t begin, end;
  int32_t parent;       // index in level l-1
  int32_t first_child;  // index in level l+1 of the first child; -1: leaf
  int32_t mask;         // octants that have a child
};

struct LvView {
  const LBox* b;
  int32_t m;
};

__host__ __device__ inline uint64_t interleave(const int64_t* cell, int dim, int level) {
  uint64_t code = 0;
  for (int bit = 0; bit < level; ++bit)
    for (int k = 0; k < dim; ++k)
      code |= static_cast<uint64_t>((cell[k] >> bit) & 1) << (dim * bit + k);
  return code;
}

__host__ __device__ inline int octant_of(const double* x, const double* c, int dim) {
  // points on a split plane go to the upper child (tree.cpp:15-21)
  int o = 0;
  for (int k = 0; k < dim; ++k) o |= (x[k] >= c[k]) << k;
  return o;
}

__device__ __forceinline__ unsigned long long ord_enc(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}

double ord_dec(unsigned long long e) {
  const uint64_t u = (e >> 63) ? (e & ~(1ull << 63)) : ~e;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

__global__ void k_bbox(const double* __restrict__ pts, int64_t n, int dim, unsigned long long* lo,
                       unsigned long long* hi) {
  unsigned long long l[3] = {~0ull, ~0ull, ~0ull}, h[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < dim; ++k) {
      const unsigned long long e = ord_enc(pts[i * dim + k]);
      l[k] = e < l[k] ? e : l[k];
      h[k] = e > h[k] ? e : h[k];
    }
  for (int k = 0; k < dim; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, l[k], o);
      const unsigned long long b = __shfl_xor_sync(0xffffffffu, h[k], o);
      l[k] = a < l[k] ? a : l[k];
      h[k] = b > h[k] ? b : h[k];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(lo + k, l[k]);
      atomicMax(hi + k, h[k]);
    }
  }
}

__global__ void k_iota(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_flag_split(const LBox* __restrict__ b, int32_t m, int cap, int at_max,
                             int32_t* flag, int* err) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int f = b[i].end - b[i].begin > cap;
  flag[i] = f;
  if (f && at_max) atomicExch(err, 1);
}

__global__ void k_split_sizes(const LBox* __restrict__ b, const int32_t* __restrict__ S, int32_t ms,
                              int64_t* sz) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ms) sz[s] = b[S[s]].end - b[S[s]].begin;
  if (s == ms) sz[s] = 0;
}

// key = (rank of the split box << 3) | octant, value = original point index
__global__ void k_keys(const LBox* __restrict__ b, const int32_t* __restrict__ S,
                       const int64_t* __restrict__ off, int32_t ms, int64_t T,
                       const int32_t* __restrict__ perm, const double* __restrict__ pts, int dim,
                       uint32_t* key, int32_t* val, int32_t* cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < T;
       j += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = ms - 1;
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    const LBox& bx = b[S[lo]];
    const int32_t p = perm[bx.begin + (j - off[lo])];
    double x[3];
    for (int k = 0; k < dim; ++k) x[k] = pts[(int64_t)p * dim + k];
    const int o = octant_of(x, bx.c, dim);
    key[j] = ((uint32_t)lo << 3) | (uint32_t)o;
    val[j] = p;
    atomicAdd(cnt + (int64_t)lo * 8 + o, 1);
  }
}

__global__ void k_scatter(const LBox* __restrict__ b, const int32_t* __restrict__ S,
                          const int64_t* __restrict__ off, int64_t T, const uint32_t* __restrict__ key,
                          const int32_t* __restrict__ val, int32_t* perm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < T;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = (int32_t)(key[j] >> 3);
    perm[b[S[s]].begin + (j - off[s])] = val[j];
  }
}

__global__ void k_nonempty(const int32_t* __restrict__ cnt, int64_t n, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = i < n && cnt[i] > 0;
}

// Non-empty children of split box s, in octant order (tree.cpp make_children).
__global__ void k_children(LBox* b, const int32_t* __restrict__ S, int32_t ms,
                           const int32_t* __restrict__ cnt, const int32_t* __restrict__ cpos,
                           LBox* nb, int dim) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ms) return;
  LBox& p = b[S[s]];
  int mask = 0, first = -1;
  int32_t off = p.begin;
  for (int c = 0; c < (1 << dim); ++c) {
    const int32_t n = cnt[(int64_t)s * 8 + c];
    if (n == 0) continue;
    const int32_t id = cpos[(int64_t)s * 8 + c];
    if (first < 0) first = id;
    mask |= 1 << c;
    LBox ch;
    ch.parent = S[s];
    ch.morton = (p.morton << dim) | (uint64_t)c;
    ch.half = p.half * 0.5;
    for (int k = 0; k < 3; ++k) {
      ch.c[k] = p.c[k];
      ch.cell[k] = 0;
    }
    for (int k = 0; k < dim; ++k) {
      const int bit = (c >> k) & 1;
      ch.cell[k] = p.cell[k] * 2 + bit;
      ch.c[k] += bit ? ch.half : -ch.half;
    }
    ch.begin = off;
    ch.end = off + n;
    off = ch.end;
    ch.first_child = -1;
    ch.mask = 0;
    nb[id] = ch;
  }
  p.first_child = first;
  p.mask = mask;
}

// Coincident points inside one leaf (they always share a leaf).
__global__ void k_dup(const LBox* __restrict__ b, const int32_t* __restrict__ perm,
                      const double* __restrict__ pts, int dim, int* found) {
  const LBox bx = b[blockIdx.x];
  if (bx.first_child >= 0) return;
  const int32_t n = bx.end - bx.begin;
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double* pi = pts + (int64_t)perm[bx.begin + i] * dim;
    for (int32_t j = i + 1; j < n; ++j) {
      const double* pj = pts + (int64_t)perm[bx.begin + j] * dim;
      bool same = true;
      for (int k = 0; k < dim; ++k) same = same && pi[k] == pj[k];
      if (same) {
        atomicExch(found, 1);
        return;
      }
    }
  }
}

__device__ int32_t find_in_level(const LvView& v, uint64_t code) {
  int32_t lo = 0, hi = v.m;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (v.b[mid].morton < code) lo = mid + 1;
    else hi = mid;
  }
  return (lo < v.m && v.b[lo].morton == code) ? lo : -1;
}

// Leaves of level l that violate 2:1 balance in the refined tree
// (the check of tree.cpp balance, without the splits).
__global__ void k_violations(const LvView* __restrict__ lv, int l, int dim, uint8_t* viol) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= lv[l].m) return;
  const LBox bx = lv[l].b[i];
  viol[i] = 0;
  if (bx.first_child >= 0) return;
  const int64_t lim = int64_t{1} << l;
  const int zr = dim == 3 ? 1 : 0;
  for (int dz = -zr; dz <= zr; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const int64_t nc[3] = {bx.cell[0] + dx, bx.cell[1] + dy, bx.cell[2] + dz};
        bool inside = true;
        for (int k = 0; k < dim; ++k) inside = inside && nc[k] >= 0 && nc[k] < lim;
        if (!inside) continue;
        for (int lvl = l; lvl >= 1; --lvl) {
          const int sh = l - lvl;
          const int64_t cc[3] = {nc[0] >> sh, nc[1] >> sh, nc[2] >> sh};
          const int32_t idx = find_in_level(lv[lvl], interleave(cc, dim, lvl));
          if (idx < 0) continue;
          if (lv[lvl].b[idx].first_child < 0 && lvl <= l - 2) {
            viol[i] = 1;
            return;
          }
          break;  // only the deepest covering box matters
        }
      }
}

// ---- neighbor lists on the final (level-major, Morton-sorted) boxes -------
struct NbArgs {
  int dim;
  int32_t nb;
  const int32_t* level_begin;
  const uint64_t* morton;
  const int64_t* cell;
  const int32_t* level;
  const uint8_t* leaf;
  const int32_t* parent;
  const int32_t* child;
  const int64_t* coll_off;
  const int32_t* coll;
};

__device__ int32_t find_box(const NbArgs& a, int lvl, uint64_t code) {
  int32_t lo = a.level_begin[lvl], hi = a.level_begin[lvl + 1];
  const int32_t end = hi;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a.morton[mid] < code) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && a.morton[lo] == code) ? lo : -1;
}

// colleagues (self included), ascending (tree.cpp build_neighbors)
__global__ void k_colleagues(NbArgs a, int64_t* count, const int64_t* off, int32_t* out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nb) return;
  const int l = a.level[i];
  const int64_t lim = int64_t{1} << l;
  const int zr = a.dim == 3 ? 1 : 0;
  int32_t ids[27];
  int n = 0;
  for (int dz = -zr; dz <= zr; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t nc[3] = {a.cell[3 * (int64_t)i] + dx, a.cell[3 * (int64_t)i + 1] + dy,
                               a.cell[3 * (int64_t)i + 2] + dz};
        bool inside = true;
        for (int k = 0; k < a.dim; ++k) inside = inside && nc[k] >= 0 && nc[k] < lim;
        if (!inside) continue;
        const int32_t id = find_box(a, l, interleave(nc, a.dim, l));
        if (id >= 0) ids[n++] = id;
      }
  if (!out) {
    count[i] = n;
    return;
  }
  for (int x = 1; x < n; ++x) {  // insertion sort, <= 27 entries
    const int32_t v = ids[x];
    int y = x - 1;
    while (y >= 0 && ids[y] > v) {
      ids[y + 1] = ids[y];
      --y;
    }
    ids[y + 1] = v;
  }
  for (int x = 0; x < n; ++x) out[off[i] + x] = ids[x];
}

// coarse: leaf colleagues of the parent (ascending as the parent's list)
__global__ void k_coarse(NbArgs a, int64_t* count, const int64_t* off, int32_t* out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nb) return;
  int64_t n = 0;
  if (a.level[i] >= 1) {
    const int32_t p = a.parent[i];
    for (int64_t e = a.coll_off[p]; e < a.coll_off[p + 1]; ++e) {
      const int32_t c = a.coll[e];
      if (!a.leaf[c]) continue;
      if (out) out[off[i] + n] = c;
      ++n;
    }
  }
  if (!out) count[i] = n;
}

// fine: children of the colleagues of a leaf, ascending
__global__ void k_fine(NbArgs a, int64_t* count, const int64_t* off, int32_t* out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nb) return;
  int64_t n = 0;
  if (a.leaf[i]) {
    for (int64_t e = a.coll_off[i]; e < a.coll_off[i + 1]; ++e) {
      const int32_t c = a.coll[e];
      for (int o = 0; o < 8; ++o) {
        const int32_t g = a.child[8 * (int64_t)c + o];
        if (g < 0) continue;
        if (out) out[off[i] + n] = g;
        ++n;
      }
    }
    if (out)
      for (int64_t x = 1; x < n; ++x) {
        int32_t* o = out + off[i];
        const int32_t v = o[x];
        int64_t y = x - 1;
        while (y >= 0 && o[y] > v) {
          o[y + 1] = o[y];
          --y;
        }
        o[y + 1] = v;
      }
  }
  if (!out) count[i] = n;
}

__global__ void k_gather_pts(const double* __restrict__ pts, const int32_t* __restrict__ perm,
                             int64_t n, int dim, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < dim; ++k) out[i * dim + k] = pts[(int64_t)perm[i] * dim + k];
}

int blocks(int64_t n, int t) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, 148 * 64)); }

// ---- host side ----------------------------------------------------------

// The reference's duplicate check (tree.cpp:160): lexicographic sort, first
// adjacent coincident pair.  Runs only to word the error.
void host_reject_duplicates(int dim, int64_t n, const double* pts) {
  std::vector<int32_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
    const double *pa = pts + (int64_t)a * dim, *pb = pts + (int64_t)b * dim;
    for (int k = 0; k < dim; ++k) {
      if (pa[k] < pb[k]) return true;
      if (pa[k] > pb[k]) return false;
    }
    return a < b;
  });
  for (int64_t i = 0; i + 1 < n; ++i) {
    const double *pa = pts + (int64_t)ord[i] * dim, *pb = pts + (int64_t)ord[i + 1] * dim;
    bool same = true;
    for (int k = 0; k < dim; ++k) same = same && pa[k] == pb[k];
    if (same)
      throw TreeFail{SFMM_EDUPLICATE, "build_tree: points " + std::to_string(ord[i]) + " and " +
                                          std::to_string(ord[i + 1]) + " coincide"};
  }
}

struct HBox {
  int32_t parent = -1;
  int32_t child[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  int32_t level = 0;
  uint64_t morton = 0;
  int64_t cell[3] = {0, 0, 0};
  double center[3] = {0, 0, 0};
  double half = 0;
  int32_t begin = 0, end = 0;
  bool leaf = false;
};

inline uint64_t level_key(int dim, int level, uint64_t code) {
  return (uint64_t{1} << (dim * level)) | code;
}

// The reference's 2:1 balance queue (tree.cpp:211-263), seeded with the
// leaves that violate it after refinement (see the file comment).
void replay_balance(std::vector<HBox>& A, std::vector<int32_t>& perm, const double* pts, int dim,
                    const std::vector<int32_t>& seeds) {
  std::unordered_map<uint64_t, int32_t> cells;
  cells.reserve(A.size() * 2);
  for (int32_t id = 0; id < (int32_t)A.size(); ++id)
    cells.emplace(level_key(dim, A[id].level, A[id].morton), id);
  std::vector<int32_t> scratch;
  std::vector<uint8_t> oct;
  auto split = [&](int32_t id, std::vector<int32_t>& out) {
    const HBox p = A[id];
    const int32_t n = p.end - p.begin;
    int32_t counts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    oct.resize(n);
    scratch.resize(n);
    for (int32_t i = 0; i < n; ++i) {
      const int o = octant_of(pts + (int64_t)perm[p.begin + i] * dim, p.center, dim);
      oct[i] = (uint8_t)o;
      ++counts[o];
    }
    int32_t pos[8], acc = 0;
    for (int c = 0; c < 8; ++c) {
      pos[c] = acc;
      acc += counts[c];
    }
    for (int32_t i = 0; i < n; ++i) scratch[pos[oct[i]]++] = perm[p.begin + i];
    std::copy(scratch.begin(), scratch.begin() + n, perm.begin() + p.begin);
    A[id].leaf = false;
    int32_t off = p.begin;
    for (int c = 0; c < (1 << dim); ++c) {
      if (counts[c] == 0) continue;
      HBox ch;
      ch.parent = id;
      ch.level = p.level + 1;
      ch.morton = (p.morton << dim) | static_cast<uint64_t>(c);
      ch.half = p.half * 0.5;
      for (int k = 0; k < 3; ++k) ch.center[k] = p.center[k];
      for (int k = 0; k < dim; ++k) {
        const int bit = (c >> k) & 1;
        ch.cell[k] = p.cell[k] * 2 + bit;
        ch.center[k] += bit ? ch.half : -ch.half;
      }
      ch.begin = off;
      ch.end = off + counts[c];
      off = ch.end;
      ch.leaf = true;
      const int32_t cid = (int32_t)A.size();
      A.push_back(ch);
      A[id].child[c] = cid;
      cells.emplace(level_key(dim, ch.level, ch.morton), cid);
      out.push_back(cid);
    }
  };
  std::deque<int32_t> work(seeds.begin(), seeds.end());
  std::vector<int32_t> created;
  const int zr = dim == 3 ? 1 : 0;
  while (!work.empty()) {
    const int32_t id = work.front();
    work.pop_front();
    if (!A[id].leaf) continue;
    for (bool again = true; again;) {
      again = false;
      const HBox box = A[id];
      if (box.level < 2) break;
      const int64_t lim = int64_t{1} << box.level;
      for (int dz = -zr; dz <= zr; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            const int64_t nc[3] = {box.cell[0] + dx, box.cell[1] + dy, box.cell[2] + dz};
            bool inside = true;
            for (int k = 0; k < dim; ++k) inside = inside && nc[k] >= 0 && nc[k] < lim;
            if (!inside) continue;
            for (int lvl = box.level; lvl >= 1; --lvl) {
              const int sh = box.level - lvl;
              const int64_t cc[3] = {nc[0] >> sh, nc[1] >> sh, nc[2] >> sh};
              const auto it = cells.find(level_key(dim, lvl, interleave(cc, dim, lvl)));
              if (it == cells.end()) continue;
              const HBox& cov = A[it->second];
              if (cov.leaf && cov.level <= box.level - 2) {
                created.clear();
                split(it->second, created);
                for (int32_t c : created) work.push_back(c);
                again = true;
              }
              break;
            }
          }
    }
  }
}

struct Timer {
  bool on = std::getenv("SFMM_TREE_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    ck(cudaDeviceSynchronize(), "sync");
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gpu tree] %-14s %.4f s\n", what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

void build(int dim, int64_t n, const double* pts_host, int cap, sfmm_gpu_tree& R) {
  if (dim != 2 && dim != 3) throw TreeFail{SFMM_EINVAL, "build_tree: dim must be 2 or 3"};
  if (cap < 1) throw TreeFail{SFMM_EINVAL, "build_tree: leaf capacity must be positive"};
  if (n < 1) throw TreeFail{SFMM_EINVAL, "build_tree: empty point set"};
  if (n > std::numeric_limits<int32_t>::max() / 2)
    throw TreeFail{SFMM_EINVAL, "build_tree: point count out of range"};
  Timer tv;
  {
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < n * dim; ++i) bad |= !std::isfinite(pts_host[i]);
    if (bad) throw TreeFail{SFMM_EINVAL, "build_tree: non-finite coordinate"};
  }
  tv.mark("validate");
  Timer tm;
  const int max_depth = dim == 2 ? kMaxDepth2 : kMaxDepth3;
  Dev<double> pts;
  pts.upload(pts_host, (size_t)n * dim);
  Dev<int32_t> perm(n);
  k_iota<<<blocks(n, 256), 256>>>(perm.p, n);
  // root box (tree.cpp:181-186)
  LBox root{};
  {
    Dev<unsigned long long> lh(6);
    std::vector<unsigned long long> init = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    ck(cudaMemcpy(lh.p, init.data(), 6 * 8, cudaMemcpyHostToDevice), "H2D");
    k_bbox<<<blocks(n, 256), 256>>>(pts.p, n, dim, lh.p, lh.p + 3);
    ck(cudaGetLastError(), "bbox");
    lh.download(init.data(), 6);
    root.half = 0;
    for (int k = 0; k < dim; ++k) {
      const double lo = ord_dec(init[k]), hi = ord_dec(init[3 + k]);
      root.c[k] = 0.5 * (lo + hi);
      root.half = std::max(root.half, 0.5 * (hi - lo));
    }
    root.half *= 1.0 + 1e-12;  // boundary points strictly inside
    if (root.half == 0.0) root.half = 0.5;
    root.begin = 0;
    root.end = (int32_t)n;
    root.parent = -1;
    root.first_child = -1;
  }
  tm.mark("upload+root");

  // ---- refinement ----
  std::vector<Dev<LBox>> L;
  std::vector<int32_t> cnt_l;
  L.emplace_back(1);
  ck(cudaMemcpy(L[0].p, &root, sizeof(LBox), cudaMemcpyHostToDevice), "H2D");
  cnt_l.push_back(1);
  Dev<uint32_t> key(n), key2(n);
  Dev<int32_t> val(n), val2(n);
  Dev<int32_t> flag, S, nsel(1), cnt, cflag, cpos;
  Dev<int64_t> sz, off;
  Dev<int> err(1);
  ck(cudaMemset(err.p, 0, sizeof(int)), "memset");
  Dev<unsigned char> temp;
  auto ensure_temp = [&](size_t bytes) {  // never NULL: CUB reads NULL as a size query
    if (bytes > temp.n || !temp.p) temp.alloc(bytes);
  };
  for (int l = 0;; ++l) {
    const int32_t m = cnt_l[l];
    flag.grow(m);
    S.grow(m);
    k_flag_split<<<(m + 255) / 256, 256>>>(L[l].p, m, cap, l == max_depth, flag.p, err.p);
    size_t tb = 0;
    cub::CountingInputIterator<int32_t> it(0);
    ck(cub::DeviceSelect::Flagged(nullptr, tb, it, flag.p, S.p, nsel.p, m), "select");
    ensure_temp(tb);
    ck(cub::DeviceSelect::Flagged(temp.p, tb, it, flag.p, S.p, nsel.p, m), "select");
    const int32_t ms = nsel.get(0);
    if (ms == 0) break;
    if (err.get(0)) {
      // the reference rejects duplicates before refining (tree.cpp:160)
      host_reject_duplicates(dim, n, pts_host);
      throw TreeFail{SFMM_EDEPTH, "build_tree: leaf capacity unreachable at depth " +
                                      std::to_string(max_depth) + " (near-duplicate points?)"};
    }
    sz.grow(ms + 1);
    off.grow(ms + 1);
    k_split_sizes<<<(ms + 1 + 255) / 256, 256>>>(L[l].p, S.p, ms, sz.p);
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, sz.p, off.p, ms + 1), "scan");
    ensure_temp(tb);
    ck(cub::DeviceScan::ExclusiveSum(temp.p, tb, sz.p, off.p, ms + 1), "scan");
    const int64_t T = off.get(ms);
    cnt.grow((size_t)ms * 8);
    ck(cudaMemset(cnt.p, 0, (size_t)ms * 8 * sizeof(int32_t)), "memset");
    k_keys<<<blocks(T, 256), 256>>>(L[l].p, S.p, off.p, ms, T, perm.p, pts.p, dim, key.p, val.p,
                                    cnt.p);
    int end_bit = 3;
    while ((int64_t{1} << (end_bit - 3)) < ms) ++end_bit;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, val.p, val2.p, T, 0, end_bit),
       "sort");
    ensure_temp(tb);
    ck(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.p, key2.p, val.p, val2.p, T, 0, end_bit),
       "sort");
    k_scatter<<<blocks(T, 256), 256>>>(L[l].p, S.p, off.p, T, key2.p, val2.p, perm.p);
    const int64_t nc = (int64_t)ms * 8;
    cflag.grow(nc + 1);
    cpos.grow(nc + 1);
    k_nonempty<<<blocks(nc + 1, 256), 256>>>(cnt.p, nc, cflag.p);
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cflag.p, cpos.p, nc + 1), "scan");
    ensure_temp(tb);
    ck(cub::DeviceScan::ExclusiveSum(temp.p, tb, cflag.p, cpos.p, nc + 1), "scan");
    const int32_t m_next = cpos.get(nc);
    L.emplace_back(m_next);
    cnt_l.push_back(m_next);
    k_children<<<(ms + 255) / 256, 256>>>(L[l].p, S.p, ms, cnt.p, cpos.p, L[l + 1].p, dim);
    ck(cudaGetLastError(), "refine");
  }
  const int D = (int)L.size() - 1;
  tm.mark("refine");

  // ---- duplicates: leaf-local ----
  if (cap <= kDupLeafMax) {
    ck(cudaMemset(err.p, 0, sizeof(int)), "memset");
    for (int l = 0; l <= D; ++l)
      k_dup<<<cnt_l[l], 128>>>(L[l].p, perm.p, pts.p, dim, err.p);
    ck(cudaGetLastError(), "duplicates");
    if (err.get(0)) host_reject_duplicates(dim, n, pts_host);
  } else {
    host_reject_duplicates(dim, n, pts_host);
  }
  tm.mark("duplicates");

  // ---- balance: violating leaves after refinement ----
  std::vector<LvView> views(D + 1);
  for (int l = 0; l <= D; ++l) views[l] = {L[l].p, cnt_l[l]};
  Dev<LvView> dviews;
  dviews.upload(views.data(), views.size());
  std::vector<int32_t> level_begin(D + 2, 0);
  for (int l = 0; l <= D; ++l) level_begin[l + 1] = level_begin[l] + cnt_l[l];
  const int32_t nb0 = level_begin[D + 1];
  std::vector<int32_t> seeds;
  {
    Dev<uint8_t> viol(nb0);
    ck(cudaMemset(viol.p, 0, nb0), "memset");
    for (int l = 2; l <= D; ++l)
      k_violations<<<(cnt_l[l] + 127) / 128, 128>>>(dviews.p, l, dim, viol.p + level_begin[l]);
    ck(cudaGetLastError(), "violations");
    std::vector<uint8_t> v(nb0, 0);
    viol.download(v.data(), nb0);
    for (int32_t i = 0; i < nb0; ++i)
      if (v[i]) seeds.push_back(i);  // level-major, Morton within a level
    if (tm.on) std::fprintf(stderr, "[gpu tree] %zu leaves violate 2:1 after refinement\n", seeds.size());
  }
  tm.mark("balance check");

  // ---- boxes to the host in (level, Morton) order ----
  std::vector<LBox> lb(nb0);
  for (int l = 0; l <= D; ++l) L[l].download(lb.data() + level_begin[l], cnt_l[l]);
  std::vector<HBox> A(nb0);
  for (int l = 0; l <= D; ++l)
    for (int32_t i = 0; i < cnt_l[l]; ++i) {
      const LBox& s = lb[level_begin[l] + i];
      HBox& h = A[level_begin[l] + i];
      h.parent = l > 0 ? level_begin[l - 1] + s.parent : -1;
      h.level = l;
      h.morton = s.morton;
      for (int k = 0; k < 3; ++k) {
        h.cell[k] = s.cell[k];
        h.center[k] = s.c[k];
      }
      h.half = s.half;
      h.begin = s.begin;
      h.end = s.end;
      h.leaf = s.first_child < 0;
      int r = 0;
      for (int c = 0; c < 8; ++c)
        if (s.mask >> c & 1) h.child[c] = level_begin[l + 1] + s.first_child + r++;
    }
  R.perm.resize(n);
  if (!seeds.empty()) {
    // order-dependent splits: the reference's sequential queue on the host
    perm.download(R.perm.data(), n);
    replay_balance(A, R.perm, pts_host, dim, seeds);
    const int32_t nb = (int32_t)A.size();
    std::vector<int32_t> order(nb);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return A[a].level != A[b].level ? A[a].level < A[b].level : A[a].morton < A[b].morton;
    });
    std::vector<int32_t> newid(nb);
    for (int32_t i = 0; i < nb; ++i) newid[order[i]] = i;
    std::vector<HBox> B(nb);
    for (int32_t i = 0; i < nb; ++i) {
      HBox b = A[order[i]];
      if (b.parent >= 0) b.parent = newid[b.parent];
      for (int32_t& c : b.child)
        if (c >= 0) c = newid[c];
      B[i] = b;
    }
    A.swap(B);
    perm.upload(R.perm.data(), n);
  } else {
    perm.download(R.perm.data(), n);
  }
  tm.mark("balance replay");

  // ---- final arrays ----
  const int32_t nb = (int32_t)A.size();
  int depth = 0;
  for (const HBox& b : A) depth = std::max(depth, b.level);
  R.dim = dim;
  R.depth = depth;
  R.leaf_cap = cap;
  R.n = n;
  R.level_begin.assign(depth + 2, 0);
  for (const HBox& b : A) ++R.level_begin[b.level + 1];
  for (int l = 0; l <= depth; ++l) R.level_begin[l + 1] += R.level_begin[l];
  R.parent.resize(nb);
  R.child.resize((size_t)nb * 8);
  R.level.resize(nb);
  R.morton.resize(nb);
  R.cell.resize((size_t)nb * 3);
  R.center.resize((size_t)nb * 3);
  R.half.resize(nb);
  R.begin.resize(nb);
  R.end.resize(nb);
  R.leaf.resize(nb);
  for (int32_t i = 0; i < nb; ++i) {
    const HBox& b = A[i];
    R.parent[i] = b.parent;
    for (int c = 0; c < 8; ++c) R.child[8 * (size_t)i + c] = b.child[c];
    R.level[i] = b.level;
    R.morton[i] = b.morton;
    for (int k = 0; k < 3; ++k) {
      R.cell[3 * (size_t)i + k] = b.cell[k];
      R.center[3 * (size_t)i + k] = b.center[k];
    }
    R.half[i] = b.half;
    R.begin[i] = b.begin;
    R.end[i] = b.end;
    R.leaf[i] = b.leaf ? 1 : 0;
  }

  // ---- neighbor lists on the device ----
  Dev<int32_t> d_lb, d_level, d_parent, d_child;
  Dev<uint64_t> d_morton;
  Dev<int64_t> d_cell;
  Dev<uint8_t> d_leaf;
  d_lb.upload(R.level_begin.data(), R.level_begin.size());
  d_level.upload(R.level.data(), nb);
  d_parent.upload(R.parent.data(), nb);
  d_child.upload(R.child.data(), R.child.size());
  d_morton.upload(R.morton.data(), nb);
  d_cell.upload(R.cell.data(), R.cell.size());
  d_leaf.upload(R.leaf.data(), nb);
  NbArgs a{};
  a.dim = dim;
  a.nb = nb;
  a.level_begin = d_lb.p;
  a.morton = d_morton.p;
  a.cell = d_cell.p;
  a.level = d_level.p;
  a.leaf = d_leaf.p;
  a.parent = d_parent.p;
  a.child = d_child.p;
  Dev<int64_t> count(nb + 1), coll_off(nb + 1), coarse_off(nb + 1), fine_off(nb + 1);
  auto csr = [&](auto kernel, Dev<int64_t>& o, std::vector<int64_t>& h_off,
                 std::vector<int32_t>& h_list) {
    ck(cudaMemset(count.p, 0, (nb + 1) * sizeof(int64_t)), "memset");
    kernel<<<(nb + 127) / 128, 128>>>(a, count.p, nullptr, nullptr);
    size_t tb = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, count.p, o.p, nb + 1), "scan");
    ensure_temp(tb);
    ck(cub::DeviceScan::ExclusiveSum(temp.p, tb, count.p, o.p, nb + 1), "scan");
    const int64_t total = o.get(nb);
    Dev<int32_t> list(total);
    kernel<<<(nb + 127) / 128, 128>>>(a, nullptr, o.p, list.p);
    ck(cudaGetLastError(), "neighbors");
    h_off.resize(nb + 1);
    o.download(h_off.data(), nb + 1);
    h_list.resize(total);
    list.download(h_list.data(), total);
    return list;
  };
  Dev<int32_t> coll = csr(k_colleagues, coll_off, R.coll_off, R.coll);
  a.coll_off = coll_off.p;
  a.coll = coll.p;
  csr(k_coarse, coarse_off, R.coarse_off, R.coarse);
  csr(k_fine, fine_off, R.fine_off, R.fine);
  tm.mark("neighbors");

  // ---- tree-order coordinates (host gather: cheaper than a 24 B/point D2H) ----
  R.pts.resize((size_t)n * dim);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < dim; ++k) R.pts[i * dim + k] = pts_host[(int64_t)R.perm[i] * dim + k];
  tm.mark("pts");
}

}  // namespace

extern "C" {

int sfmm_gpu_build_tree(int dim, int64_t n, const double* pts, int leaf_cap, int device,
                        sfmm_gpu_tree** out) {
  using sfmm_gpu::set_last_error;
  if (!out || (!pts && n > 0)) return set_last_error(SFMM_EINVAL, "build_tree: null argument");
  *out = nullptr;
  auto* R = new sfmm_gpu_tree();
  try {
    DeviceGuard device_guard(device);
    const auto t0 = std::chrono::steady_clock::now();
    build(dim, n, pts, leaf_cap, *R);
    R->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = R;
    return SFMM_OK;
  } catch (const TreeFail& f) {
    delete R;
    return set_last_error(f.code, f.msg);
  } catch (const std::bad_alloc&) {
    delete R;
    return set_last_error(SFMM_ENOMEM, "build_tree: host allocation failed");
  }
}

int sfmm_gpu_tree_arrays(const sfmm_gpu_tree* t, sfmm_tree_arrays* a) {
  if (!t || !a) return sfmm_gpu::set_last_error(SFMM_EINVAL, "tree_arrays: null argument");
  a->dim = t->dim;
  a->depth = t->depth;
  a->leaf_cap = t->leaf_cap;
  a->n_boxes = (int32_t)t->level.size();
  a->n_points = t->n;
  a->perm = t->perm.data();
  a->pts = t->pts.data();
  a->level_begin = t->level_begin.data();
  a->box_parent = t->parent.data();
  a->box_child = t->child.data();
  a->box_level = t->level.data();
  a->box_morton = t->morton.data();
  a->box_cell = t->cell.data();
  a->box_center = t->center.data();
  a->box_half = t->half.data();
  a->box_begin = t->begin.data();
  a->box_end = t->end.data();
  a->box_leaf = t->leaf.data();
  a->coll_off = t->coll_off.data();
  a->coll = t->coll.data();
  a->coarse_off = t->coarse_off.data();
  a->coarse = t->coarse.data();
  a->fine_off = t->fine_off.data();
  a->fine = t->fine.data();
  a->seconds = t->seconds;
  return SFMM_OK;
}

void sfmm_gpu_tree_destroy(sfmm_gpu_tree* t) { delete t; }

}  // extern "C"
