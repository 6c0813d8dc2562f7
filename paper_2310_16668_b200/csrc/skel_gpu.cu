// GPU skeletonization: the device counterpart of the reference's
// build_skeletons (/root/reference/proj/src/skeleton.cpp:184-260), which
// dominates the end-to-end time once the apply runs on the GPU (84 s of
// reference precompute vs 0.1 s of apply at N=1e7).
//
// Level by level from the leaves up (the only dependency is parent <- child
// skeletons), every box of a level is one CTA:
//   1. index_vec: leaf points, or the children's skeleton ids in child order
//      (skeleton.cpp:204-218), which also fixes each child's parent_offset;
//   2. proxy matrix P(y_i, x_j) on the Lobatto proxy surface of the box scaled
//      by radius_factor (skeleton.cpp:27-66, 221-243), stacked with conj(P)
//      for complex kernels, written column-major to a device workspace;
//   3. greedy Householder column-pivoted QR, stopped once the largest residual
//      column norm is <= tol * (largest initial norm), with the dqp3 norm
//      downdate and recompute guard (skeleton.cpp:68-149); warp per column for
//      the reflector application, block reductions for pivot and norms;
//   4. T = R11^{-1} R12 by back substitution (thread per redundant column) and
//      the remap to ascending skeleton / redundant positions
//      (skeleton.cpp:153-177).
// Pivot choices are rounding sensitive, so skeletons are validated by
// accuracy (and the apply by parity on the same skeletons), not by bits.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "sfmm_gpu.h"

namespace sfmm_gpu {
int set_last_error(int code, const std::string& msg);  // sfmm_gpu.cu
}

namespace {

constexpr int kSkThreads = 256;
constexpr double kPi = 3.14159265358979323846264338327950288;

struct CudaErr {
  std::string msg;
};
void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  (void)cudaGetLastError();  // reported here; do not leak into the next call
  throw CudaErr{std::string(what) + ": " + cudaGetErrorString(e)};
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

// ---- scalar helpers (real / complex) ---------------------------------------
struct Cx {
  double re, im;
};
__device__ __forceinline__ double absq(double x) { return x * x; }
__device__ __forceinline__ double absq(Cx x) { return x.re * x.re + x.im * x.im; }
__device__ __forceinline__ double conj_(double x) { return x; }
__device__ __forceinline__ Cx conj_(Cx x) { return {x.re, -x.im}; }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ Cx mul(Cx a, Cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ Cx add(Cx a, Cx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ Cx sub(Cx a, Cx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ double scale(double a, double s) { return a * s; }
__device__ __forceinline__ Cx scale(Cx a, double s) { return {a.re * s, a.im * s}; }
__device__ __forceinline__ double divs(double a, double b) { return a / b; }
__device__ __forceinline__ Cx divs(Cx a, Cx b) {
  const double d = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
template <class S>
__device__ __forceinline__ S zero();
template <>
__device__ __forceinline__ double zero<double>() { return 0.0; }
template <>
__device__ __forceinline__ Cx zero<Cx>() { return {0.0, 0.0}; }
__device__ __forceinline__ double shfl_xor(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ Cx shfl_xor(Cx v, int o) { return {shfl_xor(v.re, o), shfl_xor(v.im, o)}; }
template <class S>
__device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add(v, shfl_xor(v, o));
  return v;
}

// kernel values from r^2 (kernel.hpp:40-71)
template <class S>
__device__ __forceinline__ S kernel_value(int kernel, double kappa, double r2);
template <>
__device__ __forceinline__ double kernel_value<double>(int kernel, double, double r2) {
  if (kernel == SFMM_LAPLACE2D) return log(r2) * (-1.0 / (4.0 * kPi));
  return 1.0 / (4.0 * kPi * sqrt(r2));
}
template <>
__device__ __forceinline__ Cx kernel_value<Cx>(int, double kappa, double r2) {
  const double r = sqrt(r2);
  double s, c;
  sincos(kappa * r, &s, &c);
  return {c / (4.0 * r), s / (4.0 * r)};
}

struct LevelArgs {
  const int32_t* boxes;      // boxes of this batch (global ids)
  const int32_t* lbox;       // their index within the level
  const int64_t* iv_off;     // level-local index_vec offsets
  const int32_t* iv;         // level-local index_vec ids
  const double* pts;
  const double* center;
  const double* half;
  const double* proxy_unit;  // np x dim, in [-1, 1]
  int np, dim, kernel, rows;
  double kappa, radius, tol;
  void* work;                // column-major rows x n per box
  const int64_t* work_off;   // per batch box, in scalars
  int32_t* colid;            // level-local, pivot order (n per box)
  int32_t* kout;             // per level box
  uint8_t* sat;
};

// One CTA per box: proxy matrix + greedy Householder CPQR (skeleton.cpp:68-149).
template <class S>
__global__ void __launch_bounds__(kSkThreads) cpqr_kernel(LevelArgs a) {
  extern __shared__ unsigned char smraw[];
  const int lb = a.lbox[blockIdx.x];
  const int b = a.boxes[blockIdx.x];
  const int64_t o = a.iv_off[lb];
  const int n = (int)(a.iv_off[lb + 1] - o);
  const int M = a.rows;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  S* A = static_cast<S*>(a.work) + a.work_off[blockIdx.x];
  double* vn1 = reinterpret_cast<double*>(smraw);
  double* vn2 = vn1 + n;
  S* v = reinterpret_cast<S*>(vn2 + n);
  int* cid = reinterpret_cast<int*>(v + M);
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ double s_val;
  __shared__ int s_idx;

  // proxy matrix (column j = point iv[j]); rows np..2np-1 hold conj(P)
  const double h = a.radius * a.half[b];
  const double* c = a.center + 3 * (int64_t)b;
  const int np = a.np;
  for (int64_t idx = tid; idx < (int64_t)np * n; idx += blockDim.x) {
    const int i = (int)(idx % np), j = (int)(idx / np);
    const double* x = a.pts + (int64_t)a.iv[o + j] * a.dim;
    double r2 = 0.0;
    for (int d = 0; d < a.dim; ++d) {
      const double y = c[d] + a.proxy_unit[i * a.dim + d] * h;
      const double dx = y - x[d];
      r2 += dx * dx;
    }
    const S g = kernel_value<S>(a.kernel, a.kappa, r2);
    A[(int64_t)j * M + i] = g;
    if (M > np) A[(int64_t)j * M + np + i] = conj_(g);
  }
  for (int j = tid; j < n; j += blockDim.x) cid[j] = j;
  __syncthreads();
  // initial column norms (warp per column)
  for (int j = warp; j < n; j += nw) {
    double s = 0.0;
    for (int i = lane; i < M; i += 32) s += absq(A[(int64_t)j * M + i]);
    s = warp_sum(s);
    if (lane == 0) vn1[j] = vn2[j] = sqrt(s);
  }
  __syncthreads();
  // thresh = tol * max norm
  {
    double m = 0.0;
    for (int j = tid; j < n; j += blockDim.x) m = fmax(m, vn1[j]);
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane == 0) red_v[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < nw; ++w) mm = fmax(mm, red_v[w]);
      s_val = a.tol * mm;
    }
    __syncthreads();
  }
  const double thresh = s_val;
  const int kmax = min(M, n);
  int k = 0;
  for (; k < kmax; ++k) {
    // pivot: largest residual norm, lowest index on ties
    double bv = -1.0;
    int bi = n;
    for (int j = k + tid; j < n; j += blockDim.x)
      if (vn1[j] > bv) {
        bv = vn1[j];
        bi = j;
      }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    __syncthreads();
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v0 = red_v[0];
      int i0 = red_i[0];
      for (int w = 1; w < nw; ++w)
        if (red_v[w] > v0 || (red_v[w] == v0 && red_i[w] < i0)) {
          v0 = red_v[w];
          i0 = red_i[w];
        }
      s_val = v0;
      s_idx = i0;
    }
    __syncthreads();
    if (!(s_val > thresh)) break;
    const int piv = s_idx;
    if (piv != k) {
      for (int i = tid; i < M; i += blockDim.x) {
        const S t = A[(int64_t)piv * M + i];
        A[(int64_t)piv * M + i] = A[(int64_t)k * M + i];
        A[(int64_t)k * M + i] = t;
      }
      if (tid == 0) {
        double t = vn1[piv];
        vn1[piv] = vn1[k];
        vn1[k] = t;
        t = vn2[piv];
        vn2[piv] = vn2[k];
        vn2[k] = t;
        const int ti = cid[piv];
        cid[piv] = cid[k];
        cid[k] = ti;
      }
    }
    __syncthreads();
    // Householder reflector of column k, rows k..M-1
    S* ckp = A + (int64_t)k * M;
    {
      double s = 0.0;
      for (int i = k + tid; i < M; i += blockDim.x) s += absq(ckp[i]);
      s = warp_sum(s);
      if (lane == 0) red_v[warp] = s;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red_v[w];
        s_val = t;
      }
      __syncthreads();
    }
    const double normx = sqrt(s_val);
    if (normx == 0.0) break;
    const S x0 = ckp[k];
    const double ax0 = sqrt(absq(x0));
    S phase;
    if constexpr (sizeof(S) == 8) {
      phase = ax0 == 0.0 ? 1.0 : x0 / ax0;
    } else {
      phase = ax0 == 0.0 ? Cx{1.0, 0.0} : Cx{x0.re / ax0, x0.im / ax0};
    }
    const S beta = scale(phase, -normx);
    for (int i = k + tid; i < M; i += blockDim.x) v[i] = i == k ? sub(x0, beta) : ckp[i];
    __syncthreads();
    double vv = 0.0;
    {
      double s = 0.0;
      for (int i = k + tid; i < M; i += blockDim.x) s += absq(v[i]);
      s = warp_sum(s);
      if (lane == 0) red_v[warp] = s;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red_v[w];
        s_val = t;
      }
      __syncthreads();
      vv = s_val;
    }
    if (tid == 0) ckp[k] = beta;
    if (vv > 0.0) {
      const double sc = 2.0 / vv;
      for (int j = k + 1 + warp; j < n; j += nw) {
        S* cj = A + (int64_t)j * M;
        S w = zero<S>();
        for (int i = k + lane; i < M; i += 32) w = add(w, mul(conj_(v[i]), cj[i]));
        w = scale(warp_sum(w), sc);
        for (int i = k + lane; i < M; i += 32) cj[i] = sub(cj[i], mul(v[i], w));
        __syncwarp();
        double nv = vn1[j];
        if (nv != 0.0) {
          const double r = sqrt(absq(cj[k]));
          double t1 = 1.0 - (r / nv) * (r / nv);
          if (t1 < 0) t1 = 0;
          const double ratio = nv / vn2[j];
          if (t1 * ratio * ratio <= 1.5e-8) {  // cancellation: recompute (dqp3 guard)
            double s = 0.0;
            for (int i = k + 1 + lane; i < M; i += 32) s += absq(cj[i]);
            s = warp_sum(s);
            if (lane == 0) vn1[j] = vn2[j] = sqrt(s);
          } else if (lane == 0) {
            vn1[j] = nv * sqrt(t1);
          }
        }
      }
    }
    __syncthreads();
  }
  for (int j = tid; j < n; j += blockDim.x) a.colid[o + j] = cid[j];
  if (tid == 0) {
    a.kout[lb] = k;
    a.sat[lb] = (k == M && n > k) ? 1 : 0;
  }
}

struct SolveArgs {
  const int32_t* boxes;
  const int32_t* lbox;
  const int64_t* iv_off;
  const int32_t* colid;
  const int32_t* kk;
  int rows;
  const void* work;
  const int64_t* work_off;
  const int64_t* sk_off;  // level-local
  int32_t* skel;          // sorted skeleton positions
  int32_t* redp;          // sorted redundant positions
  const int64_t* T_off;   // level-local, scalars
  void* T;
};

// T = R11^{-1} R12 in ascending skeleton / redundant order (skeleton.cpp:153-177).
template <class S>
__global__ void __launch_bounds__(kSkThreads) solve_kernel(SolveArgs a) {
  extern __shared__ int rank[];  // n entries: rank of each pivot-order column in its sorted set
  const int lb = a.lbox[blockIdx.x];
  const int64_t o = a.iv_off[lb];
  const int n = (int)(a.iv_off[lb + 1] - o);
  const int k = a.kk[lb], r = n - k, M = a.rows;
  const int32_t* cid = a.colid + o;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int lo = i < k ? 0 : k, hi = i < k ? k : n;
    int rk = 0;
    for (int l = lo; l < hi; ++l) rk += cid[l] < cid[i];
    rank[i] = rk;
    if (i < k)
      a.skel[a.sk_off[lb] + rk] = cid[i];
    else
      a.redp[(o - a.sk_off[lb]) + rk] = cid[i];  // red offset = iv_off - sk_off
  }
  __syncthreads();
  const S* A = static_cast<const S*>(a.work) + a.work_off[blockIdx.x];
  S* T = static_cast<S*>(a.T) + a.T_off[lb];
  for (int j = k + threadIdx.x; j < n; j += blockDim.x) {
    const int cj = rank[j];
    for (int i = k - 1; i >= 0; --i) {
      S s = A[(int64_t)j * M + i];
      for (int l = i + 1; l < k; ++l) s = sub(s, mul(A[(int64_t)l * M + i], T[(int64_t)rank[l] * r + cj]));
      T[(int64_t)rank[i] * r + cj] = divs(s, A[(int64_t)i * M + i]);
    }
  }
}

// index_vec of the boxes of one level: leaf ranges or children's skeleton ids.
__global__ void build_iv_kernel(const int32_t* boxes, int nbox, const int64_t* iv_off,
                                int32_t* iv, const uint8_t* leaf, const int32_t* begin,
                                const int32_t* child_off, const int32_t* child,
                                const int64_t* c_iv_off, const int32_t* c_iv,
                                const int64_t* c_sk_off, const int32_t* c_skel,
                                const int32_t* c_lidx, int32_t* poff) {
  const int lb = blockIdx.x;
  if (lb >= nbox) return;
  const int b = boxes[lb];
  const int64_t o = iv_off[lb];
  if (leaf[b]) {
    const int n = (int)(iv_off[lb + 1] - o);
    for (int i = threadIdx.x; i < n; i += blockDim.x) iv[o + i] = begin[b] + i;
    return;
  }
  int64_t off = 0;
  for (int e = child_off[b]; e < child_off[b + 1]; ++e) {
    const int c = child[e];
    const int cl = c_lidx[c];  // index of the child within its level
    const int64_t s0 = c_sk_off[cl], s1 = c_sk_off[cl + 1];
    for (int64_t i = threadIdx.x; i < s1 - s0; i += blockDim.x)
      iv[o + off + i] = c_iv[c_iv_off[cl] + c_skel[s0 + i]];
    if (threadIdx.x == 0) poff[c] = (int32_t)off;
    off += s1 - s0;
  }
}

std::vector<double> lobatto(int p) {
  std::vector<double> t(p);
  for (int j = 0; j <= (p - 1) / 2; ++j) {
    const double v = std::cos(kPi * j / (p - 1));
    t[j] = v;
    t[p - 1 - j] = -v;
  }
  if (p % 2 == 1) t[p / 2] = 0.0;
  return t;
}

// unit proxy surface (the reference's proxy_surface with c = 0, h = 1)
std::vector<double> unit_proxy(int dim, int edge2d, int face3d) {
  std::vector<double> out;
  if (dim == 2) {
    const auto t = lobatto(edge2d);
    for (int j = 0; j < edge2d; ++j) out.insert(out.end(), {t[j], -1.0, t[j], 1.0});
    for (int j = 1; j + 1 < edge2d; ++j) out.insert(out.end(), {-1.0, t[j], 1.0, t[j]});
  } else {
    const auto t = lobatto(face3d);
    const int g = face3d;
    for (int i = 0; i < g; ++i)
      for (int j = 0; j < g; ++j)
        for (int k = 0; k < g; ++k) {
          if (i != 0 && i != g - 1 && j != 0 && j != g - 1 && k != 0 && k != g - 1) continue;
          out.insert(out.end(), {t[i], t[j], t[k]});
        }
  }
  return out;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  void download(std::vector<T>& v, size_t count) const {
    v.resize(count);
    if (count) ck(cudaMemcpy(v.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }
};


}  // namespace

struct sfmm_skel_result {
  std::vector<int64_t> iv_off, sk_off, rd_off, T_off;
  std::vector<int32_t> iv, skel_pos, red_pos, poff;
  // interpolation operators in box order (global T_off), resident on `device`;
  // the host copy T is made on demand (sfmm_gpu_skel_fill / _describe)
  double* d_T = nullptr;
  int device = 0, sw = 1;
  // owner of d_T, shared with single-rank plans built from this result
  // (skel_share_T): the operators are not copied, and whichever of the two
  // is destroyed last frees them
  std::shared_ptr<double> T_owner;
  bool have_host_T = false;
  std::vector<double> T;
  int32_t k_max = 0, saturated = 0;
  int64_t proj = 0;
  double seconds = 0;
  sfmm_skel_result() = default;
  sfmm_skel_result(const sfmm_skel_result&) = delete;
  sfmm_skel_result& operator=(const sfmm_skel_result&) = delete;
  ~sfmm_skel_result() = default;
  size_t t_scalars() const { return T_off.empty() ? 0 : (size_t)T_off.back() * sw; }
  void ensure_host_T() {
    if (have_host_T) return;
    T.resize(t_scalars());
    if (!T.empty()) {
      DeviceGuard device_guard(device);
      ck(cudaMemcpy(T.data(), d_T, T.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H T");
    }
    have_host_T = true;
  }
};

namespace {

// mask (n_boxes, may be NULL = every box): only the boxes with mask[b] != 0
// are skeletonized; the others get an empty index_vec (n = k = 0, no T).  The
// masked boxes must form whole subtrees (a rank's share of a sharded plan,
// sfmm_gpu_build_skeletons_subset): each masked box's result depends only on
// its own subtree, so it is bit-identical to the unmasked build's.
template <class S>
void run_skeletons(const sfmm_tree_desc& t, int kernel, double kappa, double tol, double radius,
                   int edge2d, int face3d, const uint8_t* mask, sfmm_skel_result& R) {
  constexpr int SW = sizeof(S) / 8;
  const auto t_run0 = std::chrono::steady_clock::now();
  const int nb = t.n_boxes, dim = t.dim, depth = t.depth;
  const std::vector<double> unit = unit_proxy(dim, edge2d, face3d);
  const int np = (int)unit.size() / dim;
  const int rows = SW == 2 ? 2 * np : np;
  // children CSR (ascending id = child octant order)
  std::vector<int32_t> child_off(nb + 1, 0), child;
  for (int b = 1; b < nb; ++b) child_off[t.box_parent[b] + 1]++;
  for (int b = 0; b < nb; ++b) child_off[b + 1] += child_off[b];
  child.resize(child_off[nb]);
  {
    std::vector<int32_t> fill(child_off.begin(), child_off.end() - 1);
    for (int b = 1; b < nb; ++b) child[fill[t.box_parent[b]]++] = b;
  }
  std::vector<int32_t> lidx(nb);
  for (int l = 0; l <= depth; ++l)
    for (int b = t.level_begin[l]; b < t.level_begin[l + 1]; ++b) lidx[b] = b - t.level_begin[l];

  DevBuf<double> d_pts, d_center, d_half, d_unit;
  d_pts.upload(std::vector<double>(t.pts, t.pts + t.n_points * dim));
  d_center.upload(std::vector<double>(t.box_center, t.box_center + 3 * (size_t)nb));
  d_half.upload(std::vector<double>(t.box_half, t.box_half + nb));
  d_unit.upload(unit);
  DevBuf<uint8_t> d_leaf;
  d_leaf.upload(std::vector<uint8_t>(t.box_leaf, t.box_leaf + nb));
  DevBuf<int32_t> d_begin, d_child_off, d_child, d_lidx, d_poff;
  d_begin.upload(std::vector<int32_t>(t.box_begin, t.box_begin + nb));
  d_child_off.upload(child_off);
  d_child.upload(child);
  d_lidx.upload(lidx);
  d_poff.upload(std::vector<int32_t>(nb, 0));

  // per-level results (level-local offsets), kept on the device until the end
  struct Level {
    std::vector<int64_t> iv_off, sk_off, T_off;
    std::vector<int32_t> k;
    DevBuf<int64_t> d_iv_off, d_sk_off, d_T_off;
    DevBuf<int32_t> d_iv, d_skel, d_red, d_k, d_colid;
    DevBuf<double> d_T;
    std::vector<double> h_T;  // the level's T moved to the host (device memory short)
    bool T_host = false;
  };
  std::vector<Level> L(depth + 1);
  // Moves a level's operators to the host and frees the device buffer.
  auto spill = [&](Level& lv, size_t nt) {
    lv.h_T.resize(nt);
    if (nt) ck(cudaMemcpy(lv.h_T.data(), lv.d_T.p, nt * sizeof(double), cudaMemcpyDeviceToHost), "D2H T");
    cudaFree(lv.d_T.p);
    lv.d_T.p = nullptr;
    lv.d_T.n = 0;
    lv.T_host = true;
  };
#ifndef SFMM_SKEL_WORK_GB
#define SFMM_SKEL_WORK_GB 12
#endif
  const size_t work_cap = (size_t)SFMM_SKEL_WORK_GB << 30;  // proxy-matrix workspace per batch
  DevBuf<double> d_work;
  const bool verbose = std::getenv("SFMM_SKEL_VERBOSE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  if (verbose) {
    ck(cudaDeviceSynchronize(), "sync");
    std::fprintf(stderr, "[skel] setup: %.3f s\n", secs(t_run0, now()));
  }
  for (int l = depth; l >= 0; --l) {
    const auto t_lv = now();
    Level& lv = L[l];
    const int b0 = t.level_begin[l], b1 = t.level_begin[l + 1], nl = b1 - b0;
    // index_vec sizes: leaf points or the children's k
    std::vector<int64_t> n(nl);
    std::vector<int32_t> act;  // level-local indices of the boxes to skeletonize
    act.reserve(nl);
    for (int i = 0; i < nl; ++i) {
      const int b = b0 + i;
      if (mask && !mask[b]) {
        n[i] = 0;
        continue;
      }
      act.push_back(i);
      if (t.box_leaf[b]) {
        n[i] = t.box_end[b] - t.box_begin[b];
      } else {
        int64_t s = 0;
        for (int e = child_off[b]; e < child_off[b + 1]; ++e) s += L[l + 1].k[lidx[child[e]]];
        n[i] = s;
      }
    }
    lv.iv_off.assign(nl + 1, 0);
    for (int i = 0; i < nl; ++i) lv.iv_off[i + 1] = lv.iv_off[i] + n[i];
    lv.d_iv_off.upload(lv.iv_off);
    lv.d_iv.alloc(lv.iv_off[nl]);
    std::vector<int32_t> boxes(nl);
    std::iota(boxes.begin(), boxes.end(), b0);
    DevBuf<int32_t> d_boxes;
    d_boxes.upload(boxes);
    {
      const Level* cl = l < depth ? &L[l + 1] : nullptr;
      build_iv_kernel<<<nl, 128>>>(d_boxes.p, nl, lv.d_iv_off.p, lv.d_iv.p, d_leaf.p, d_begin.p,
                                   d_child_off.p, d_child.p, cl ? cl->d_iv_off.p : nullptr,
                                   cl ? cl->d_iv.p : nullptr, cl ? cl->d_sk_off.p : nullptr,
                                   cl ? cl->d_skel.p : nullptr, d_lidx.p, d_poff.p);
      ck(cudaGetLastError(), "build_iv");
    }
    lv.k.assign(nl, 0);
    if (l < 2) {  // level-1 boxes interact densely; no compression
      lv.sk_off.assign(nl + 1, 0);
      lv.T_off.assign(nl + 1, 0);
      lv.d_sk_off.upload(lv.sk_off);
      lv.d_skel.alloc(0);
      lv.d_red.alloc(0);
      lv.d_T.alloc(0);
      continue;
    }
    lv.d_k.alloc(nl);
    lv.d_colid.alloc(lv.iv_off[nl]);
    DevBuf<uint8_t> d_sat;
    d_sat.alloc(nl);
    // CPQR in batches bounded by the workspace
    std::vector<int64_t> woff(nl + 1, 0);
    for (int i = 0; i < nl; ++i) woff[i + 1] = woff[i] + (int64_t)rows * n[i];
    int64_t nmax = 0;
    for (int i = 0; i < nl; ++i) nmax = std::max<int64_t>(nmax, n[i]);
    const size_t smem = nmax * (2 * sizeof(double) + sizeof(int)) + rows * sizeof(S) + 64;
    if (smem > 200 * 1024) throw CudaErr{"box too large for the GPU skeletonizer"};
    ck(cudaFuncSetAttribute(cpqr_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
       "smem attr");
    // T sizes need k: run CPQR for the whole level (batched), then solve
    // batches: consecutive runs of `act` (positions into it)
    const int na = (int)act.size();
    std::vector<int> batch_start{0};
    {
      int64_t acc = 0;
      for (int a = 0; a < na; ++a) {
        const int64_t sz = (int64_t)rows * n[act[a]] * sizeof(S);
        if (acc > 0 && acc + sz > (int64_t)work_cap) {
          batch_start.push_back(a);
          acc = 0;
        }
        acc += sz;
      }
      batch_start.push_back(na);
    }
    // the solve needs R of every box, so the level's workspace must persist
    // until its solve: process batch by batch (CPQR, k, solve)
    lv.sk_off.assign(nl + 1, 0);
    lv.T_off.assign(nl + 1, 0);
    std::vector<int32_t> kk_all(nl, 0);
    std::vector<uint8_t> sat_all(nl, 0);
    // first pass: CPQR + solve need level-wide sk_off/T_off, so run CPQR for
    // all batches first, keeping R only for the batch being solved; the
    // workspace is reused, so each batch is factored and solved before the next
    int filled = 0;  // level-local boxes whose sk_off / T_off prefix is final
    for (size_t bi = 0; bi + 1 < batch_start.size() && na > 0; ++bi) {
      const int a0 = batch_start[bi], a1 = batch_start[bi + 1];
      const int cnt = a1 - a0;
      // the batch's boxes are level-local indices act[a0..a1); their
      // workspaces are packed in that order
      std::vector<int64_t> wo(cnt);
      std::vector<int32_t> lb(cnt), bx(cnt);
      int64_t wsum = 0;
      for (int a = 0; a < cnt; ++a) {
        const int i = act[a0 + a];
        wo[a] = wsum;  // in scalars S
        wsum += woff[i + 1] - woff[i];
        lb[a] = i;
        bx[a] = boxes[i];
      }
      DevBuf<int64_t> d_wo;
      d_wo.upload(wo);
      const size_t wbytes = (size_t)wsum * sizeof(S);
      if (d_work.n * sizeof(double) < wbytes) d_work.alloc(wbytes / sizeof(double) + 1);
      DevBuf<int32_t> d_lb, d_bx;
      d_lb.upload(lb);
      d_bx.upload(bx);
      LevelArgs a{};
      a.boxes = d_bx.p;
      a.lbox = d_lb.p;
      a.iv_off = lv.d_iv_off.p;
      a.iv = lv.d_iv.p;
      a.pts = d_pts.p;
      a.center = d_center.p;
      a.half = d_half.p;
      a.proxy_unit = d_unit.p;
      a.np = np;
      a.dim = dim;
      a.kernel = kernel;
      a.rows = rows;
      a.kappa = kappa;
      a.radius = radius;
      a.tol = tol;
      a.work = d_work.p;
      a.work_off = d_wo.p;
      a.colid = lv.d_colid.p;
      a.kout = lv.d_k.p;
      a.sat = d_sat.p;
      cpqr_kernel<S><<<cnt, kSkThreads, smem>>>(a);
      ck(cudaGetLastError(), "cpqr");
      {
        std::vector<int32_t> kd(nl);
        const int i_lo = act[a0], i_hi = act[a1 - 1] + 1;
        ck(cudaMemcpy(kd.data() + i_lo, lv.d_k.p + i_lo, (i_hi - i_lo) * sizeof(int32_t),
                      cudaMemcpyDeviceToHost),
           "D2H k");
        for (int a = a0; a < a1; ++a) kk_all[act[a]] = kd[act[a]];
        // level-local offsets are prefix sums in box order; batches run in
        // order, skipped boxes contribute nothing
        for (int i = filled; i < i_hi; ++i) {
          lv.sk_off[i + 1] = lv.sk_off[i] + kk_all[i];
          lv.T_off[i + 1] = lv.T_off[i] + (int64_t)kk_all[i] * (n[i] - kk_all[i]);
        }
        filled = i_hi;
      }
      // grow the level outputs to this batch's end and solve it
      if (bi == 0) {
        // upper bounds for the whole level: k <= n, k*r <= n^2/4
        int64_t kcap = 0, tcap = 0;
        for (int i = 0; i < nl; ++i) {
          kcap += std::min<int64_t>(n[i], rows);
          tcap += (n[i] / 2) * ((n[i] + 1) / 2);
        }
        lv.d_skel.alloc(kcap);
        lv.d_red.alloc(lv.iv_off[nl]);
        lv.d_T.alloc((size_t)tcap * SW);
        lv.d_sk_off.alloc(nl + 1);
        lv.d_T_off.alloc(nl + 1);
      }
      ck(cudaMemcpy(lv.d_sk_off.p, lv.sk_off.data(), (nl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice),
         "H2D sk_off");
      ck(cudaMemcpy(lv.d_T_off.p, lv.T_off.data(), (nl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice),
         "H2D T_off");
      SolveArgs s{};
      s.boxes = d_bx.p;
      s.lbox = d_lb.p;
      s.iv_off = lv.d_iv_off.p;
      s.colid = lv.d_colid.p;
      s.kk = lv.d_k.p;
      s.rows = rows;
      s.work = d_work.p;
      s.work_off = d_wo.p;
      s.sk_off = lv.d_sk_off.p;
      s.skel = lv.d_skel.p;
      s.redp = lv.d_red.p;
      s.T_off = lv.d_T_off.p;
      s.T = lv.d_T.p;
      solve_kernel<S><<<cnt, kSkThreads, nmax * sizeof(int)>>>(s);
      ck(cudaGetLastError(), "solve");
      {
        std::vector<uint8_t> sd(nl);
        const int i_lo = act[a0], i_hi = act[a1 - 1] + 1;
        ck(cudaMemcpy(sd.data() + i_lo, d_sat.p + i_lo, (i_hi - i_lo) * sizeof(uint8_t),
                      cudaMemcpyDeviceToHost),
           "D2H sat");
        for (int a = a0; a < a1; ++a) sat_all[act[a]] = sd[act[a]];
      }
    }
    // boxes after the last skeletonized one (and every box of a level with
    // none) close the prefix sums
    for (int i = filled; i < nl; ++i) {
      lv.sk_off[i + 1] = lv.sk_off[i] + kk_all[i];
      lv.T_off[i + 1] = lv.T_off[i] + (int64_t)kk_all[i] * (n[i] - kk_all[i]);
    }
    if (na == 0) {  // nothing of this level here: empty outputs
      lv.d_skel.alloc(0);
      lv.d_red.alloc(0);
      lv.d_T.alloc(0);
      lv.d_sk_off.upload(lv.sk_off);
      lv.d_T_off.upload(lv.T_off);
    }
    ck(cudaDeviceSynchronize(), "level");
    if (verbose)
      std::fprintf(stderr, "[skel] level %d: %d boxes, %zu batches, nmax %lld, %.3f s\n", l, nl,
                   batch_start.size() - 1, (long long)nmax, secs(t_lv, now()));
    lv.k = kk_all;
    // the level's T buffer was sized for k r <= n^2/4 per box: keep only the
    // exact part (on the host when even that no longer fits, e.g. N=1e8)
    if (l >= 2) {
      const size_t nt = (size_t)lv.T_off[nl] * SW;
      static const bool force_host = std::getenv("SFMM_SKEL_HOST_STAGING") != nullptr;  // tests
      if (force_host) {
        spill(lv, nt);
      } else if (nt < lv.d_T.n) {
        double* exact = nullptr;
        if (cudaMalloc(&exact, std::max<size_t>(nt, 1) * sizeof(double)) == cudaSuccess) {
          if (nt) ck(cudaMemcpy(exact, lv.d_T.p, nt * sizeof(double), cudaMemcpyDeviceToDevice), "compact T");
          cudaFree(lv.d_T.p);
          lv.d_T.p = exact;
          lv.d_T.n = nt;
        } else {
          (void)cudaGetLastError();
          spill(lv, nt);
        }
      }
    }
    for (int i = 0; i < nl; ++i) {
      R.k_max = std::max(R.k_max, kk_all[i]);
      R.saturated += sat_all[i];
      R.proj += (int64_t)kk_all[i] * (n[i] - kk_all[i]);
    }
  }
  // assemble the global (box-order) CSR arrays on the host
  const auto t_asm = now();
  R.iv_off.assign(nb + 1, 0);
  R.sk_off.assign(nb + 1, 0);
  R.rd_off.assign(nb + 1, 0);
  R.T_off.assign(nb + 1, 0);
  for (int l = 0; l <= depth; ++l) {
    const int b0 = t.level_begin[l], nl = t.level_begin[l + 1] - b0;
    for (int i = 0; i < nl; ++i) {
      const int b = b0 + i;
      const int64_t n = L[l].iv_off[i + 1] - L[l].iv_off[i];
      const int64_t k = L[l].k[i];
      R.iv_off[b + 1] = R.iv_off[b] + n;
      R.sk_off[b + 1] = R.sk_off[b] + k;
      R.rd_off[b + 1] = R.rd_off[b] + (l >= 2 ? n - k : 0);
      R.T_off[b + 1] = R.T_off[b] + (l >= 2 ? k * (n - k) : 0);
    }
  }
  R.iv.resize(R.iv_off[nb]);
  R.skel_pos.resize(R.sk_off[nb]);
  R.red_pos.resize(R.rd_off[nb]);
  R.sw = SW;
  R.have_host_T = false;
  R.T.clear();
  ck(cudaGetDevice(&R.device), "cudaGetDevice");
  d_work.alloc(0);  // the proxy workspace is no longer needed
  // the result's T; levels still on the device move to the host (largest
  // first) until it fits
  while (cudaMalloc(&R.d_T, std::max<size_t>(R.t_scalars() + 2, 1) * sizeof(double)) != cudaSuccess) {
    (void)cudaGetLastError();
    int big = -1;
    for (int l = 2; l <= depth; ++l)
      if (!L[l].T_host && L[l].d_T.p && (big < 0 || L[l].d_T.n > L[big].d_T.n)) big = l;
    if (big < 0) {
      ck(cudaErrorMemoryAllocation, "cudaMalloc T");
      break;
    }
    spill(L[big], L[big].d_T.n);
    if (verbose) std::fprintf(stderr, "[skel] level %d operators staged on the host\n", big);
  }
  {
    const int dev = R.device;
    R.T_owner.reset(R.d_T, [dev](double* ptr) {
      int cur = -1;
      if (cudaGetDevice(&cur) != cudaSuccess) cur = -1;
      cudaSetDevice(dev);
      cudaFree(ptr);
      if (cur >= 0) cudaSetDevice(cur);
    });
  }
  for (int l = 0; l <= depth; ++l) {
    const int b0 = t.level_begin[l], nl = t.level_begin[l + 1] - b0;
    if (nl == 0) continue;
    Level& lv = L[l];
    const int64_t niv = lv.iv_off[nl];
    if (niv) ck(cudaMemcpy(R.iv.data() + R.iv_off[b0], lv.d_iv.p, niv * 4, cudaMemcpyDeviceToHost), "D2H iv");
    if (l < 2) continue;
    const int64_t nsk = lv.sk_off[nl], nt = lv.T_off[nl];
    if (nsk) ck(cudaMemcpy(R.skel_pos.data() + R.sk_off[b0], lv.d_skel.p, nsk * 4, cudaMemcpyDeviceToHost), "D2H skel");
    if (niv - nsk)
      ck(cudaMemcpy(R.red_pos.data() + R.rd_off[b0], lv.d_red.p, (niv - nsk) * 4, cudaMemcpyDeviceToHost),
         "D2H red");
    if (nt && lv.T_host)
      ck(cudaMemcpy(R.d_T + R.T_off[b0] * SW, lv.h_T.data(), nt * SW * 8, cudaMemcpyHostToDevice), "H2D T");
    else if (nt)
      ck(cudaMemcpy(R.d_T + R.T_off[b0] * SW, lv.d_T.p, nt * SW * 8, cudaMemcpyDeviceToDevice), "D2D T");
    std::vector<double>().swap(lv.h_T);
    lv.d_T.alloc(0);  // release the level's buffer early
  }
  R.poff.resize(nb);
  ck(cudaMemcpy(R.poff.data(), d_poff.p, nb * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H poff");
  if (verbose) {
    std::fprintf(stderr, "[skel] assemble: %.3f s\n", secs(t_asm, now()));
    std::fprintf(stderr, "[skel] total: %.3f s\n", secs(t_run0, now()));
  }
}

}  // namespace

extern "C" {

int sfmm_gpu_build_skeletons_subset(const sfmm_tree_desc* tree, int kernel, double kappa,
                                    double tol, double proxy_radius, int proxy_edge2d,
                                    int proxy_face3d, int device, const uint8_t* box_mask,
                                    sfmm_skel_result** out) {
  using sfmm_gpu::set_last_error;
  if (!tree || !out) return set_last_error(SFMM_EINVAL, "build_skeletons: null argument");
  *out = nullptr;
  if (box_mask)  // whole subtrees: a masked box's children are masked
    for (int32_t b = 1; b < tree->n_boxes; ++b)
      if (box_mask[tree->box_parent[b]] && !box_mask[b])
        return set_last_error(SFMM_EINVAL,
                              "build_skeletons_subset: the mask must select whole subtrees");
  if (!(tol > 0.0 && tol < 0.5))
    return set_last_error(SFMM_EINVAL, "build_skeletons: tolerance must lie in (0, 0.5)");
  if (kernel == SFMM_HELMHOLTZ2D)
    return set_last_error(SFMM_EUNSUPPORTED, "build_skeletons: helmholtz2d has no device path");
  const int want = kernel == SFMM_LAPLACE2D ? 2 : 3;
  if (tree->dim != want)
    return set_last_error(SFMM_EINVAL, "build_skeletons: kernel dimension does not match the tree");
  const double radius = proxy_radius > 0 ? proxy_radius : 2.95;
  const int edge = proxy_edge2d > 0 ? proxy_edge2d : 24;
  const int face = proxy_face3d > 0 ? proxy_face3d : 8;
  if (!(radius > 1.0) || edge < 4 || face < 4)
    return set_last_error(SFMM_EINVAL, "build_skeletons: bad proxy configuration");
  auto* R = new sfmm_skel_result();
  try {
    DeviceGuard device_guard(device);
    const auto t0 = std::chrono::steady_clock::now();
    if (kernel == SFMM_HELMHOLTZ3D)
      run_skeletons<Cx>(*tree, kernel, kappa, tol, radius, edge, face, box_mask, *R);
    else
      run_skeletons<double>(*tree, kernel, kappa, tol, radius, edge, face, box_mask, *R);
    R->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = R;
    return SFMM_OK;
  } catch (const CudaErr& e) {
    delete R;
    return set_last_error(SFMM_ECUDA, "build_skeletons: " + e.msg);
  } catch (const std::bad_alloc&) {
    delete R;
    return set_last_error(SFMM_ENOMEM, "build_skeletons: host allocation failed");
  }
}

int sfmm_gpu_build_skeletons(const sfmm_tree_desc* tree, int kernel, double kappa, double tol,
                             double proxy_radius, int proxy_edge2d, int proxy_face3d, int device,
                             sfmm_skel_result** out) {
  return sfmm_gpu_build_skeletons_subset(tree, kernel, kappa, tol, proxy_radius, proxy_edge2d,
                                         proxy_face3d, device, nullptr, out);
}

int sfmm_gpu_skel_fill(sfmm_skel_result* r, sfmm_plan_desc* d, int32_t* k_max,
                       int64_t* proj_scalars, int32_t* saturated, double* seconds) {
  return sfmm_gpu_skel_describe(r, d, 1, k_max, proj_scalars, saturated, seconds);
}

int sfmm_gpu_skel_describe(sfmm_skel_result* r, sfmm_plan_desc* d, int with_host_T,
                           int32_t* k_max, int64_t* proj_scalars, int32_t* saturated,
                           double* seconds) {
  using sfmm_gpu::set_last_error;
  if (!r || !d) return set_last_error(SFMM_EINVAL, "skel_describe: null argument");
  if (with_host_T) {
    try {
      r->ensure_host_T();
    } catch (const CudaErr& e) {
      return set_last_error(SFMM_ECUDA, "skel_describe: " + e.msg);
    } catch (const std::bad_alloc&) {
      return set_last_error(SFMM_ENOMEM, "skel_describe: host allocation failed");
    }
  }
  d->iv_off = r->iv_off.data();
  d->iv = r->iv.data();
  d->sk_off = r->sk_off.data();
  d->skel_pos = r->skel_pos.data();
  d->rd_off = r->rd_off.data();
  d->red_pos = r->red_pos.data();
  d->T_off = r->T_off.data();
  d->T = with_host_T ? r->T.data() : nullptr;
  d->box_parent_offset = r->poff.data();
  if (k_max) *k_max = r->k_max;
  if (proj_scalars) *proj_scalars = r->proj;
  if (saturated) *saturated = r->saturated;
  if (seconds) *seconds = r->seconds;
  return SFMM_OK;
}

const double* sfmm_gpu_skel_device_T(const sfmm_skel_result* r, int* device, int64_t* n_scalars) {
  if (!r) return nullptr;
  if (device) *device = r->device;
  if (n_scalars) *n_scalars = (int64_t)r->t_scalars();
  return r->d_T;
}

void sfmm_gpu_skel_destroy(sfmm_skel_result* r) { delete r; }

}  // extern "C"

namespace sfmm_gpu {
std::shared_ptr<double> skel_share_T(const sfmm_skel_result* r) {
  return r ? r->T_owner : std::shared_ptr<double>();
}
}  // namespace sfmm_gpu

extern "C" {

}  // extern "C"
