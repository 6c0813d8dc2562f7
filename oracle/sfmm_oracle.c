/*
 * TEST INFRASTRUCTURE -- CPU restatement of the reference SRS-FMM apply
 * (Algorithm 2), used only as the parity checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg.  It is never
 * linked into, called by or shipped with the product library.
 *
 * It walks the flat sfmm_plan_desc (include/sfmm_gpu.h) in exactly the
 * reference's loop order, so on the same descriptor it reproduces
 * sfmm::fmm_apply bit for bit when both are compiled without FMA contraction
 * (pinned against oracle/_ref/libsfmm_ref.so in tests/test_oracle.py).
 *
 * Reference anchors (/root/reference/proj/...):
 *   add_block          src/apply.cpp:16-42
 *   upward_pass        src/apply.cpp:109-146
 *   translate_ifo      src/apply.cpp:148-177
 *   translate_ifs      src/apply.cpp:179-208
 *   translate_tfo      src/apply.cpp:210-239
 *   level1_dense       src/apply.cpp:241-266
 *   downward_pass      src/apply.cpp:268-304
 *   fmm_apply          src/apply.cpp:306-337 (depth<2 -> direct_sum, oracle.cpp:35-49)
 *   from_r2            include/sfmm/kernel.hpp:40-71
 * Helmholtz2d (long-double Hankel, bessel.cpp) is out of scope: returns 6.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "sfmm_gpu.h"

#define ORC_PI 3.14159265358979323846264338327950288

typedef struct { double re, im; } cx;

typedef struct {
  int kernel, dim, cplx;
  double kappa;
  int coincident;
} orc_ctx;

/* from_r2 (kernel.hpp:40-71).  Real kernels return im = 0. */
static cx orc_from_r2(const orc_ctx* c, double r2) {
  cx g = {0.0, 0.0};
  switch (c->kernel) {
    case SFMM_LAPLACE2D: g.re = log(r2) * (-1.0 / (4.0 * ORC_PI)); break;
    case SFMM_LAPLACE3D: g.re = 1.0 / (4.0 * ORC_PI * sqrt(r2)); break;
    case SFMM_HELMHOLTZ3D: {
      const double r = sqrt(r2);
      const double kr = c->kappa * r;
      g.re = cos(kr) / (4.0 * r);
      g.im = sin(kr) / (4.0 * r);
      break;
    }
    default: break;
  }
  return g;
}

/* Scalars are stored as 1 (real) or 2 (complex) doubles. */
static inline void orc_mac(const orc_ctx* c, cx g, const double* q, cx* acc) {
  if (c->cplx) {
    acc->re += g.re * q[0] - g.im * q[1];
    acc->im += g.re * q[1] + g.im * q[0];
  } else {
    acc->re += g.re * q[0];
  }
}

/* add_block<kSub> (apply.cpp:16-42): u[i] +/-= sum_j G(xt_i, xs_j) q[j],
 * zero diagonal keyed on ids, coincident distinct ids flagged. */
static void orc_add_block(orc_ctx* c, int sub, const double* pts, const int32_t* ti,
                          int64_t nt, const int32_t* si, int64_t ns, const double* q,
                          double* u) {
  const int d = c->dim, w = c->cplx ? 2 : 1;
  for (int64_t i = 0; i < nt; ++i) {
    const double* xi = pts + (int64_t)ti[i] * d;
    cx acc = {0.0, 0.0};
    for (int64_t j = 0; j < ns; ++j) {
      const double* xj = pts + (int64_t)si[j] * d;
      double r2 = 0;
      for (int k = 0; k < d; ++k) {
        const double dx = xi[k] - xj[k];
        r2 += dx * dx;
      }
      if (r2 == 0.0) {
        if (ti[i] != si[j]) c->coincident = 1;
        continue;
      }
      orc_mac(c, orc_from_r2(c, r2), q + j * w, &acc);
    }
    if (sub) {
      u[i * w] -= acc.re;
      if (w == 2) u[i * w + 1] -= acc.im;
    } else {
      u[i * w] += acc.re;
      if (w == 2) u[i * w + 1] += acc.im;
    }
  }
}

/* direct_sum (oracle.cpp:9-49) on points in the given order. */
static int orc_direct(orc_ctx* c, int64_t n, const double* pts, const double* q,
                      int64_t nt, const int32_t* targets, double* u) {
  const int d = c->dim, w = c->cplx ? 2 : 1;
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t i = targets ? targets[t] : t;
    const double* xi = pts + i * d;
    cx acc = {0.0, 0.0};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double* xj = pts + j * d;
      double r2 = 0;
      for (int k = 0; k < d; ++k) {
        const double dx = xi[k] - xj[k];
        r2 += dx * dx;
      }
      if (r2 == 0.0) {
        c->coincident = 1;
        continue;
      }
      orc_mac(c, orc_from_r2(c, r2), q + j * w, &acc);
    }
    u[t * w] = acc.re;
    if (w == 2) u[t * w + 1] = acc.im;
  }
  return c->coincident ? SFMM_EDUPLICATE : SFMM_OK;
}

int oracle_direct_sum(int kernel, double kappa, int dim, int64_t n, const double* pts,
                      const double* q, int64_t nt, const int32_t* targets, double* u) {
  orc_ctx c = {kernel, dim, kernel >= SFMM_HELMHOLTZ2D, kappa, 0};
  if (kernel == SFMM_HELMHOLTZ2D) return SFMM_EUNSUPPORTED;
  return orc_direct(&c, n, pts, q, nt, targets, u);
}

/* One right-hand side.  q, u: original order, w doubles per scalar.
 * stats (may be NULL): ifo, ifs, tfo, level1 pair counts, direct_fallback. */
static int orc_apply1(const sfmm_plan_desc* D, const double* q, double* u, int64_t* stats) {
  orc_ctx c = {D->kernel, D->dim, D->kernel >= SFMM_HELMHOLTZ2D, D->kappa, 0};
  const int w = c.cplx ? 2 : 1, d = D->dim;
  const int64_t n = D->n_points, nb = D->n_boxes;
  if (D->kernel == SFMM_HELMHOLTZ2D) return SFMM_EUNSUPPORTED;
  if (stats) memset(stats, 0, 5 * sizeof(int64_t));

  if (D->depth < 2) { /* apply.cpp:316-328 */
    double* orig = (double*)malloc(sizeof(double) * n * d);
    for (int64_t t = 0; t < n; ++t)
      memcpy(orig + (int64_t)D->perm[t] * d, D->pts + t * d, sizeof(double) * d);
    int rc = orc_direct(&c, n, orig, q, n, NULL, u);
    free(orig);
    if (stats) stats[4] = 1;
    return rc;
  }

  /* make_state (apply.cpp:50-65): q,u over index_vec; qhat,uhat over skel. */
  const int64_t ns = D->iv_off[nb], nk = D->sk_off[nb];
  double* Q = (double*)calloc((size_t)(ns * w + 1), sizeof(double));
  double* U = (double*)calloc((size_t)(ns * w + 1), sizeof(double));
  double* QH = (double*)calloc((size_t)(nk * w + 1), sizeof(double));
  double* UH = (double*)calloc((size_t)(nk * w + 1), sizeof(double));
  int32_t* sid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nk + 1));
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t i = D->sk_off[b]; i < D->sk_off[b + 1]; ++i)
      sid[i] = D->iv[D->iv_off[b] + D->skel_pos[i]];

  /* children in ascending id order (octant order in the reference tree) */
  int64_t* ch_off = (int64_t*)calloc((size_t)(nb + 1), sizeof(int64_t));
  int32_t* ch = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb + 1));
  for (int64_t b = 0; b < nb; ++b)
    if (D->box_parent[b] >= 0) ch_off[D->box_parent[b] + 1]++;
  for (int64_t b = 0; b < nb; ++b) ch_off[b + 1] += ch_off[b];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb + 1));
    memcpy(fill, ch_off, sizeof(int64_t) * (size_t)(nb + 1));
    for (int64_t b = 0; b < nb; ++b)
      if (D->box_parent[b] >= 0) ch[fill[D->box_parent[b]]++] = (int32_t)b;
    free(fill);
  }

  /* upward_pass (apply.cpp:109-146) */
  for (int l = D->depth; l >= 0; --l) {
    for (int64_t b = D->level_begin[l]; b < D->level_begin[l + 1]; ++b) {
      double* qb = Q + D->iv_off[b] * w;
      if (D->box_leaf[b]) {
        const int64_t np = D->box_end[b] - D->box_begin[b];
        for (int64_t i = 0; i < np; ++i)
          memcpy(qb + i * w, q + (int64_t)D->perm[D->box_begin[b] + i] * w, sizeof(double) * w);
      } else {
        for (int64_t e = ch_off[b]; e < ch_off[b + 1]; ++e) {
          const int32_t cb = ch[e];
          const int64_t kc = D->sk_off[cb + 1] - D->sk_off[cb];
          memcpy(qb + (int64_t)D->box_parent_offset[cb] * w, QH + D->sk_off[cb] * w,
                 sizeof(double) * w * kc);
        }
      }
      if (l < 2) continue;
      const int64_t k = D->sk_off[b + 1] - D->sk_off[b];
      const int64_t r = D->rd_off[b + 1] - D->rd_off[b];
      double* qh = QH + D->sk_off[b] * w;
      const int32_t* sp = D->skel_pos + D->sk_off[b];
      const int32_t* rp = D->red_pos + D->rd_off[b];
      for (int64_t i = 0; i < k; ++i) memcpy(qh + i * w, qb + (int64_t)sp[i] * w, sizeof(double) * w);
      const double* T = D->T + D->T_off[b] * w;
      for (int64_t i = 0; i < k; ++i) {
        cx acc = {0.0, 0.0};
        for (int64_t j = 0; j < r; ++j) {
          const double* t = T + (i * r + j) * w;
          const double* x = qb + (int64_t)rp[j] * w;
          if (w == 2) {
            acc.re += t[0] * x[0] - t[1] * x[1];
            acc.im += t[0] * x[1] + t[1] * x[0];
          } else {
            acc.re += t[0] * x[0];
          }
        }
        qh[i * w] += acc.re;
        if (w == 2) qh[i * w + 1] += acc.im;
      }
    }
  }

  int64_t n_ifo = 0, n_ifs = 0, n_tfo = 0, n_l1 = 0;
#define IVB(b) (D->iv + D->iv_off[b])
#define NB(b) (D->iv_off[(b) + 1] - D->iv_off[b])
#define KB(b) (D->sk_off[(b) + 1] - D->sk_off[b])
  /* translate_ifo (apply.cpp:148-177) */
  for (int l = 2; l <= D->depth; ++l)
    for (int64_t b = D->level_begin[l]; b < D->level_begin[l + 1]; ++b)
      for (int64_t e = D->coll_off[b]; e < D->coll_off[b + 1]; ++e) {
        const int32_t cb = D->coll[e];
        ++n_ifo;
        orc_add_block(&c, 0, D->pts, IVB(b), NB(b), IVB(cb), NB(cb), Q + D->iv_off[cb] * w,
                      U + D->iv_off[b] * w);
        orc_add_block(&c, 1, D->pts, sid + D->sk_off[b], KB(b), sid + D->sk_off[cb], KB(cb),
                      QH + D->sk_off[cb] * w, UH + D->sk_off[b] * w);
      }
  /* translate_ifs (apply.cpp:179-208) */
  for (int l = 2; l <= D->depth; ++l)
    for (int64_t b = D->level_begin[l]; b < D->level_begin[l + 1]; ++b)
      for (int64_t e = D->coarse_off[b]; e < D->coarse_off[b + 1]; ++e) {
        const int32_t cb = D->coarse[e];
        ++n_ifs;
        orc_add_block(&c, 0, D->pts, IVB(b), NB(b), IVB(cb), NB(cb), Q + D->iv_off[cb] * w,
                      U + D->iv_off[b] * w);
        orc_add_block(&c, 1, D->pts, sid + D->sk_off[b], KB(b), IVB(cb), NB(cb),
                      Q + D->iv_off[cb] * w, UH + D->sk_off[b] * w);
      }
  /* translate_tfo (apply.cpp:210-239) */
  for (int64_t b = 0; b < nb; ++b) {
    if (!D->box_leaf[b] || D->box_level[b] < 1) continue;
    for (int64_t e = D->fine_off[b]; e < D->fine_off[b + 1]; ++e) {
      const int32_t cb = D->fine[e];
      ++n_tfo;
      orc_add_block(&c, 0, D->pts, IVB(b), NB(b), IVB(cb), NB(cb), Q + D->iv_off[cb] * w,
                    U + D->iv_off[b] * w);
      orc_add_block(&c, 1, D->pts, IVB(b), NB(b), sid + D->sk_off[cb], KB(cb),
                    QH + D->sk_off[cb] * w, U + D->iv_off[b] * w);
    }
  }
  /* level1_dense (apply.cpp:241-266) */
  {
    const int lev = D->depth >= 1 ? 1 : 0;
    for (int64_t b = D->level_begin[lev]; b < D->level_begin[lev + 1]; ++b)
      for (int64_t cb = D->level_begin[lev]; cb < D->level_begin[lev + 1]; ++cb) {
        ++n_l1;
        orc_add_block(&c, 0, D->pts, IVB(b), NB(b), IVB(cb), NB(cb), Q + D->iv_off[cb] * w,
                      U + D->iv_off[b] * w);
      }
  }
  /* downward_pass (apply.cpp:268-304) */
  for (int l = 2; l <= D->depth; ++l)
    for (int64_t b = D->level_begin[l]; b < D->level_begin[l + 1]; ++b) {
      const int64_t k = KB(b), r = D->rd_off[b + 1] - D->rd_off[b];
      double* uh = UH + D->sk_off[b] * w;
      const double* up = U + (D->iv_off[D->box_parent[b]] + D->box_parent_offset[b]) * w;
      for (int64_t i = 0; i < k * w; ++i) uh[i] += up[i];
      double* ub = U + D->iv_off[b] * w;
      const int32_t* sp = D->skel_pos + D->sk_off[b];
      const int32_t* rp = D->red_pos + D->rd_off[b];
      for (int64_t i = 0; i < k; ++i) {
        ub[(int64_t)sp[i] * w] += uh[i * w];
        if (w == 2) ub[(int64_t)sp[i] * w + 1] += uh[i * w + 1];
      }
      const double* T = D->T + D->T_off[b] * w;
      for (int64_t i = 0; i < k; ++i) {
        const double* ui = uh + i * w;
        for (int64_t j = 0; j < r; ++j) {
          const double* t = T + (i * r + j) * w;
          double* o = ub + (int64_t)rp[j] * w;
          if (w == 2) { /* conj(t) * u */
            o[0] += t[0] * ui[0] + t[1] * ui[1];
            o[1] += t[0] * ui[1] - t[1] * ui[0];
          } else {
            o[0] += t[0] * ui[0];
          }
        }
      }
    }
  for (int64_t b = 0; b < nb; ++b) {
    if (!D->box_leaf[b]) continue;
    const int64_t np = D->box_end[b] - D->box_begin[b];
    for (int64_t i = 0; i < np; ++i)
      memcpy(u + (int64_t)D->perm[D->box_begin[b] + i] * w, U + (D->iv_off[b] + i) * w,
             sizeof(double) * w);
  }
#undef IVB
#undef NB
#undef KB
  free(Q); free(U); free(QH); free(UH); free(sid); free(ch_off); free(ch);
  if (stats) {
    stats[0] = n_ifo; stats[1] = n_ifs; stats[2] = n_tfo; stats[3] = n_l1; stats[4] = 0;
  }
  return c.coincident ? SFMM_EDUPLICATE : SFMM_OK;
}

/* nrhs columns, column-major, each column an independent apply. */
int oracle_fmm_apply(const sfmm_plan_desc* D, const double* q, double* u, int nrhs,
                     int64_t* stats) {
  const int w = D->kernel >= SFMM_HELMHOLTZ2D ? 2 : 1;
  for (int r = 0; r < nrhs; ++r) {
    int rc = orc_apply1(D, q + (int64_t)r * D->n_points * w, u + (int64_t)r * D->n_points * w,
                        r == 0 ? stats : NULL);
    if (rc) return rc;
  }
  return SFMM_OK;
}
