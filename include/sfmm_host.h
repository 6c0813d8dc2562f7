/*
 * sfmm_host.h -- host-side container of a plan descriptor built on the GPU.
 *
 * The precompute that feeds the apply (tree, neighbor lists, skeletons) runs
 * on the device (sfmm_gpu_build_tree / sfmm_gpu_build_skeletons, SURVEY.md
 * 8(f)); a C++ caller of the reference keeps using the reference's own
 * sfmm::build_tree / build_neighbor_lists / build_skeletons
 * (/root/reference/proj/src/tree.cpp:148-355, skeleton.cpp:184-260) and the
 * drop-in header include/sfmm_gpu.hpp.  This small library only holds the
 * host copies of those device results as one sfmm_plan_desc
 * (include/sfmm_gpu.h) and provides the benchmark's synthetic inputs
 *   sfmm::generate_points / generate_charges(_complex)
 *                               /root/reference/proj/src/bench.cpp:102-161
 * plus the clustered Gaussian of config 3(b).
 */
#ifndef SFMM_HOST_H_
#define SFMM_HOST_H_

#include <stdint.h>

#include "sfmm_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: sfmm_gpu.h (SFMM_EDEPTH = sfmm::DepthExceededError). */

/* Distributions, same order as sfmm::Distribution (bench.hpp:15), plus the
 * clustered Gaussian of config 3(b), which the reference does not define. */
enum {
  SFMM_DIST_SQUARE = 0,
  SFMM_DIST_ANNULUS = 1,
  SFMM_DIST_CUBE = 2,
  SFMM_DIST_SPHERE = 3,
  SFMM_DIST_GAUSSIAN = 4
};

/* sfmm::ProxyConfig (skeleton.hpp:13-17); zero fields take the defaults
 * 2.95 / 24 / 8. */
typedef struct sfmm_proxy_config {
  double radius_factor;
  int32_t edge_points_2d;
  int32_t face_grid_3d;
} sfmm_proxy_config;

typedef struct sfmm_host_info {
  int32_t depth;
  int32_t n_boxes;
  int64_t n_leaves;
  int32_t k_max;
  int32_t saturated_boxes;
  int64_t proj_scalars;     /* SkeletonSet::proj_scalars */
  double t_tree;            /* seconds: build_tree + build_neighbor_lists */
  double t_skel;            /* seconds: build_skeletons */
} sfmm_host_info;

typedef struct sfmm_host_plan sfmm_host_plan;

int sfmm_host_generate_points(int dist, int64_t n, uint64_t seed, double* out);
int sfmm_host_generate_charges(int64_t n, uint64_t seed, double* out);
int sfmm_host_generate_charges_complex(int64_t n, uint64_t seed, double* out);

/* Flat view of the plan; valid until sfmm_host_destroy. */
const sfmm_plan_desc* sfmm_host_desc(sfmm_host_plan* plan);

/* Box geometry (centre: n_boxes*3, half-width: n_boxes), needed by the GPU
 * skeletonizer's proxy surfaces (sfmm_tree_desc in sfmm_gpu.h). */
int sfmm_host_box_geometry(const sfmm_host_plan* plan, double* center, double* half);

/* Host plan around a tree built elsewhere (e.g. sfmm_gpu_build_tree): the
 * arrays are copied; skeletons can then be set (sfmm_host_set_skeletons). */
int sfmm_host_adopt_tree(const sfmm_tree_arrays* tree, sfmm_host_plan** out);

/* Replaces the plan's skeleton fields with externally built ones (e.g. from
 * sfmm_gpu_build_skeletons); the arrays are copied.  skel->T may be NULL: the
 * interpolation operators then live only on the device (the plan's desc.T is
 * NULL until sfmm_host_set_T). */
int sfmm_host_set_skeletons(sfmm_host_plan* plan, const sfmm_plan_desc* skel, int kernel,
                            double kappa, int32_t k_max, int64_t proj_scalars, int32_t saturated,
                            double t_skel);

/* Sets (copies) the interpolation operators: n_scalars doubles, box order,
 * matching the plan's T_off (interleaved complex for Helmholtz). */
int sfmm_host_set_T(sfmm_host_plan* plan, const double* T, int64_t n_scalars);

int sfmm_host_info_get(const sfmm_host_plan* plan, sfmm_host_info* info);

void sfmm_host_destroy(sfmm_host_plan* plan);

/* Number of OpenMP threads the host-side copies use (0 keeps the default). */
void sfmm_host_set_threads(int n);
int sfmm_host_get_threads(void);

const char* sfmm_host_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SFMM_HOST_H_ */
