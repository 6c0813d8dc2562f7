// Skeletonization (Algorithm 1): proxy-surface interpolative decompositions,
// level by level from the leaves up.
//
// Follows /root/reference/proj/src/skeleton.cpp: proxy surface on the box
// scaled by radius_factor (:27-66), proxy matrix P(y_i, x_j) from the kernel,
// stacked with its conjugate for complex kernels (:221-243), greedy
// column-pivoted QR stopped at eps * (largest initial column norm) with a
// dqp3-style norm downdate (:68-149), T = R11^{-1} R12 (:153-162), skeleton
// and redundant positions sorted ascending (:164-177).  Boxes above level 2
// only receive index vectors.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <numeric>

#include "host.h"

namespace sfmm_host {
namespace {

using cplx = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;

inline double abs2(double x) { return x * x; }
inline double abs2(const cplx& x) { return x.real() * x.real() + x.imag() * x.imag(); }
inline double conj_s(double x) { return x; }
inline cplx conj_s(const cplx& x) { return std::conj(x); }

std::vector<double> lobatto(int p) {
  std::vector<double> t(p);
  for (int j = 0; j <= (p - 1) / 2; ++j) {
    const double v = std::cos(kPi * j / (p - 1));
    t[j] = v;
    t[p - 1 - j] = -v;  // mirrored so opposite faces coincide bit for bit
  }
  if (p % 2 == 1) t[p / 2] = 0.0;
  return t;
}

std::vector<double> proxy_points(int dim, const double* c, double half, const Proxy& px) {
  if (!(px.radius_factor > 1.0)) throw std::invalid_argument("proxy_surface: radius factor must exceed 1");
  std::vector<double> out;
  const double h = px.radius_factor * half;
  if (dim == 2) {
    const int p = px.edge_points_2d;
    if (p < 4) throw std::invalid_argument("proxy_surface: need at least 4 nodes per edge");
    const auto t = lobatto(p);
    for (int j = 0; j < p; ++j) {
      out.insert(out.end(), {c[0] + t[j] * h, c[1] - h, c[0] + t[j] * h, c[1] + h});
    }
    for (int j = 1; j + 1 < p; ++j) {
      out.insert(out.end(), {c[0] - h, c[1] + t[j] * h, c[0] + h, c[1] + t[j] * h});
    }
  } else {
    const int g = px.face_grid_3d;
    if (g < 4) throw std::invalid_argument("proxy_surface: need at least a 4x4 face grid");
    const auto t = lobatto(g);
    for (int i = 0; i < g; ++i)
      for (int j = 0; j < g; ++j)
        for (int k = 0; k < g; ++k) {
          const bool surface = i == 0 || i == g - 1 || j == 0 || j == g - 1 || k == 0 || k == g - 1;
          if (!surface) continue;
          out.insert(out.end(), {c[0] + t[i] * h, c[1] + t[j] * h, c[2] + t[k] * h});
        }
  }
  return out;
}

template <class S>
S kernel_value(int kernel, double kappa, double r2);

template <>
double kernel_value<double>(int kernel, double, double r2) {
  if (kernel == 0) return std::log(r2) * (-1.0 / (4.0 * kPi));
  return 1.0 / (4.0 * kPi * std::sqrt(r2));
}

template <>
cplx kernel_value<cplx>(int, double kappa, double r2) {
  const double r = std::sqrt(r2);
  const double kr = kappa * r;
  return {std::cos(kr) / (4.0 * r), std::sin(kr) / (4.0 * r)};
}

}  // namespace

// Greedy column-pivoted Householder QR on a column-major m x n matrix (copied),
// stopped once every residual column norm is <= eps * max initial norm.
template <class S>
int column_id(const S* a_in, int64_t m, int64_t n, double eps, std::vector<int32_t>& skel,
              std::vector<int32_t>& red, std::vector<S>& interp) {
  skel.clear();
  red.clear();
  interp.clear();
  if (n == 0) return 0;
  std::vector<S> A(a_in, a_in + m * n);
  std::vector<int32_t> col(n);
  std::iota(col.begin(), col.end(), 0);
  std::vector<double> nrm(n), nrm_ref(n);
  double nmax = 0;
  for (int64_t j = 0; j < n; ++j) {
    double s = 0;
    const S* cj = A.data() + j * m;
    for (int64_t i = 0; i < m; ++i) s += abs2(cj[i]);
    nrm[j] = nrm_ref[j] = std::sqrt(s);
    nmax = std::max(nmax, nrm[j]);
  }
  const double thresh = eps * nmax;
  const int64_t kmax = std::min(m, n);
  std::vector<S> v(m);
  int64_t k = 0;
  for (; k < kmax; ++k) {
    int64_t piv = k;
    for (int64_t j = k + 1; j < n; ++j)
      if (nrm[j] > nrm[piv]) piv = j;  // lowest index wins ties
    if (!(nrm[piv] > thresh)) break;
    if (piv != k) {
      std::swap_ranges(A.begin() + piv * m, A.begin() + (piv + 1) * m, A.begin() + k * m);
      std::swap(nrm[piv], nrm[k]);
      std::swap(nrm_ref[piv], nrm_ref[k]);
      std::swap(col[piv], col[k]);
    }
    S* ck = A.data() + k * m;
    double sq = 0;
    for (int64_t i = k; i < m; ++i) sq += abs2(ck[i]);
    const double alpha = std::sqrt(sq);
    if (alpha == 0.0) break;
    const S x0 = ck[k];
    const double ax0 = std::sqrt(abs2(x0));
    const S phase = ax0 == 0.0 ? S(1) : S(x0 / ax0);
    const S beta = -phase * alpha;
    // reflector v = x - beta e_k, applied as I - 2 v v^H / (v^H v)
    double vv = 0;
    v[k] = x0 - beta;
    vv += abs2(v[k]);
    for (int64_t i = k + 1; i < m; ++i) {
      v[i] = ck[i];
      vv += abs2(v[i]);
    }
    ck[k] = beta;
    if (vv > 0) {
      const double sc = 2.0 / vv;
      for (int64_t j = k + 1; j < n; ++j) {
        S* cj = A.data() + j * m;
        S w{};
        for (int64_t i = k; i < m; ++i) w += conj_s(v[i]) * cj[i];
        w *= sc;
        for (int64_t i = k; i < m; ++i) cj[i] -= v[i] * w;
        if (nrm[j] != 0.0) {
          const double rk = std::sqrt(abs2(cj[k]));
          double f = 1.0 - (rk / nrm[j]) * (rk / nrm[j]);
          if (f < 0) f = 0;
          const double ratio = nrm[j] / nrm_ref[j];
          if (f * ratio * ratio <= 1.5e-8) {  // cancellation: recompute (dqp3 guard)
            double s = 0;
            for (int64_t i = k + 1; i < m; ++i) s += abs2(cj[i]);
            nrm[j] = nrm_ref[j] = std::sqrt(s);
          } else {
            nrm[j] *= std::sqrt(f);
          }
        }
      }
    }
  }
  const int64_t r = n - k;
  // X = R11^{-1} R12 by back substitution, X is k x r (column j = rhs j)
  std::vector<S> X((size_t)(k * r));
  for (int64_t j = 0; j < r; ++j) {
    const S* rhs = A.data() + (k + j) * m;
    for (int64_t i = k - 1; i >= 0; --i) {
      S s = rhs[i];
      for (int64_t l = i + 1; l < k; ++l) s -= A[l * m + i] * X[l * r + j];
      X[i * r + j] = s / A[i * m + i];
    }
  }
  skel.assign(col.begin(), col.begin() + k);
  red.assign(col.begin() + k, col.end());
  std::vector<int32_t> srank(k), rrank(r);
  {
    std::vector<int32_t> o(k);
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int32_t a, int32_t b) { return skel[a] < skel[b]; });
    for (int64_t i = 0; i < k; ++i) srank[o[i]] = (int32_t)i;
    std::vector<int32_t> p(r);
    std::iota(p.begin(), p.end(), 0);
    std::sort(p.begin(), p.end(), [&](int32_t a, int32_t b) { return red[a] < red[b]; });
    for (int64_t j = 0; j < r; ++j) rrank[p[j]] = (int32_t)j;
  }
  interp.assign((size_t)(k * r), S{});
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < r; ++j) interp[(size_t)srank[i] * r + rrank[j]] = X[i * r + j];
  std::sort(skel.begin(), skel.end());
  std::sort(red.begin(), red.end());
  return (int)k;
}

template int column_id<double>(const double*, int64_t, int64_t, double, std::vector<int32_t>&,
                               std::vector<int32_t>&, std::vector<double>&);
template int column_id<cplx>(const cplx*, int64_t, int64_t, double, std::vector<int32_t>&,
                             std::vector<int32_t>&, std::vector<cplx>&);

namespace {

template <class S>
Skeletons skeletonize(const Tree& t, int kernel, double kappa, double tol, const Proxy& px) {
  constexpr bool kCplx = std::is_same<S, cplx>::value;
  const int dim = t.dim;
  const int32_t nb = (int32_t)t.boxes.size();
  struct Per {
    std::vector<int32_t> iv, sk, rd;
    std::vector<S> T;
    int32_t poff = 0;
    bool saturated = false;
  };
  std::vector<Per> per(nb);
  for (int l = t.depth; l >= 0; --l) {
    const int32_t b0 = t.level_begin[l], b1 = t.level_begin[l + 1];
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t b = b0; b < b1; ++b) {
      const Box& box = t.boxes[b];
      Per& pb = per[b];
      if (box.leaf) {
        pb.iv.resize(box.npoints());
        std::iota(pb.iv.begin(), pb.iv.end(), box.begin);
      } else {
        int32_t off = 0;  // children's skeletons in octant order (skeleton.cpp:207-217)
        for (int32_t c : box.child) {
          if (c < 0) continue;
          per[c].poff = off;
          for (int32_t pos : per[c].sk) pb.iv.push_back(per[c].iv[pos]);
          off += (int32_t)per[c].sk.size();
        }
      }
      if (l < 2) continue;  // level-1 boxes interact densely
      const int64_t nc = (int64_t)pb.iv.size();
      const std::vector<double> prx = proxy_points(dim, box.center, box.half, px);
      const int64_t np = (int64_t)prx.size() / dim;
      const int64_t rows = kCplx ? 2 * np : np;
      std::vector<S> P((size_t)(rows * nc));  // column-major
      for (int64_t j = 0; j < nc; ++j) {
        const double* x = t.pts.data() + (int64_t)pb.iv[j] * dim;
        S* cj = P.data() + j * rows;
        for (int64_t i = 0; i < np; ++i) {
          const double* y = prx.data() + i * dim;
          double r2 = 0;
          for (int d = 0; d < dim; ++d) {
            const double dx = y[d] - x[d];
            r2 += dx * dx;
          }
          const S v = kernel_value<S>(kernel, kappa, r2);
          cj[i] = v;
          if constexpr (kCplx) cj[np + i] = conj_s(v);
        }
      }
      const int k = column_id<S>(P.data(), rows, nc, tol, pb.sk, pb.rd, pb.T);
      pb.saturated = k == rows && nc > k;
    }
  }
  Skeletons s;
  const int sw = kCplx ? 2 : 1;
  s.iv_off.assign(nb + 1, 0);
  s.sk_off.assign(nb + 1, 0);
  s.rd_off.assign(nb + 1, 0);
  s.T_off.assign(nb + 1, 0);
  s.parent_offset.resize(nb);
  for (int32_t b = 0; b < nb; ++b) {
    s.iv_off[b + 1] = s.iv_off[b] + (int64_t)per[b].iv.size();
    s.sk_off[b + 1] = s.sk_off[b] + (int64_t)per[b].sk.size();
    s.rd_off[b + 1] = s.rd_off[b] + (int64_t)per[b].rd.size();
    s.T_off[b + 1] = s.T_off[b] + (int64_t)per[b].T.size();
    s.parent_offset[b] = per[b].poff;
    s.k_max = std::max(s.k_max, (int)per[b].sk.size());
    s.saturated += per[b].saturated ? 1 : 0;
    s.proj_scalars += (int64_t)per[b].sk.size() * (int64_t)per[b].rd.size();
  }
  s.iv.resize(s.iv_off[nb]);
  s.skel_pos.resize(s.sk_off[nb]);
  s.red_pos.resize(s.rd_off[nb]);
  s.T.resize((size_t)s.T_off[nb] * sw);
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t b = 0; b < nb; ++b) {
    Per& p = per[b];
    std::copy(p.iv.begin(), p.iv.end(), s.iv.begin() + s.iv_off[b]);
    std::copy(p.sk.begin(), p.sk.end(), s.skel_pos.begin() + s.sk_off[b]);
    std::copy(p.rd.begin(), p.rd.end(), s.red_pos.begin() + s.rd_off[b]);
    if (!p.T.empty())
      std::memcpy(s.T.data() + s.T_off[b] * sw, p.T.data(), sizeof(S) * p.T.size());
    std::vector<S>().swap(p.T);
  }
  return s;
}

}  // namespace

Skeletons build_skeletons(const Tree& t, int kernel, double kappa, double tol, const Proxy& px) {
  if (!(tol > 0.0 && tol < 0.5))
    throw std::invalid_argument("build_skeletons: tolerance must lie in (0, 0.5)");
  const int want = (kernel == 0 || kernel == 2) ? 2 : 3;
  if (t.dim != want)
    throw std::invalid_argument("build_skeletons: kernel dimension does not match the tree");
  if (kernel == 2) throw std::logic_error("helmholtz2d has no device apply path");
  if (kernel == 3) return skeletonize<cplx>(t, kernel, kappa, tol, px);
  return skeletonize<double>(t, kernel, kappa, tol, px);
}

}  // namespace sfmm_host
