// TEST INFRASTRUCTURE -- exercises the C++ drop-in include/sfmm_gpu.hpp the way
// a reference user would: the reference's own pipeline (build_tree,
// build_neighbor_lists, build_skeletons, make_plan), then the CPU
// sfmm::fmm_apply and the GPU sfmm::gpu::fmm_apply on the same plan and
// charges.  Prints one line per case and exits non-zero if any case misses
// rel-l2 1e-12 or the ApplyStats differ.  Built by oracle/Makefile into
// oracle/_ref/dropin_parity (links the reference objects and libsfmm_gpu.so).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sfmm/apply.hpp"
#include "sfmm/bench.hpp"
#include "sfmm/oracle.hpp"
#include "sfmm_gpu.hpp"

using namespace sfmm;

template <class T>
double rel_l2(const std::vector<T>& u, const std::vector<T>& r) {
  double num = 0, den = 0;
  for (size_t i = 0; i < u.size(); ++i) {
    num += abs_sq(u[i] - r[i]);
    den += abs_sq(r[i]);
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

static std::vector<int> g_devices = {0, 0, 0, 0};  // argv[1]: comma-separated ids

template <class K>
int run(const char* name, const K& kern, Distribution dist, int64_t n, int leaf, double tol) {
  using S = typename K::scalar;
  const PointSet pts = generate_points(dist, n, 1);
  const Tree tree = build_tree(pts, leaf);
  const NeighborLists nb = build_neighbor_lists(tree);
  const SkeletonSet<S> skel = build_skeletons(tree, kern, tol);
  const ApplyPlan<K> plan = make_plan(kern, tree, nb, skel);
  std::vector<S> q;
  if constexpr (std::is_same_v<S, double>)
    q = generate_charges(n, 2);
  else
    q = generate_charges_complex(n, 2);
  ApplyStats s_cpu, s_gpu;
  const std::vector<S> u_cpu = fmm_apply(plan, q, &s_cpu);
  gpu::GpuPlan<K> gplan(plan);
  const std::vector<S> u_gpu = gpu::fmm_apply(gplan, q, &s_gpu);
  const double err = rel_l2(u_gpu, u_cpu);
  const bool stats_ok = s_cpu.n_ifo_pairs == s_gpu.n_ifo_pairs &&
                        s_cpu.n_ifs_pairs == s_gpu.n_ifs_pairs &&
                        s_cpu.n_tfo_pairs == s_gpu.n_tfo_pairs &&
                        s_cpu.n_level1_pairs == s_gpu.n_level1_pairs &&
                        s_cpu.direct_fallback == s_gpu.direct_fallback;
  const bool ok = err <= 1e-12 && stats_ok;
  std::printf("%-28s n=%-7lld depth=%d rel_l2=%.3e stats=%s %s\n", name, (long long)n, tree.depth,
              err, stats_ok ? "same" : "DIFFER", ok ? "OK" : "FAIL");
  // the same plan sharded over g_devices in this process: exchanges inside
  // the library (peer copies), result within 1e-12 of the reference
  ApplyStats s_multi;
  gpu::GpuPlan<K> gmulti(plan, g_devices);
  const std::vector<S> u_multi = gpu::fmm_apply(gmulti, q, &s_multi);
  const double err_multi = rel_l2(u_multi, u_cpu);
  const bool multi_ok = err_multi <= 1e-12 && s_multi.n_ifo_pairs == s_cpu.n_ifo_pairs &&
                        s_multi.n_ifs_pairs == s_cpu.n_ifs_pairs &&
                        s_multi.n_tfo_pairs == s_cpu.n_tfo_pairs &&
                        s_multi.n_level1_pairs == s_cpu.n_level1_pairs;
  std::printf("%-28s %zu-rank plan rel_l2 vs CPU %.3e %s\n", name, g_devices.size(), err_multi,
              multi_ok ? "OK" : "FAIL");
  // the reference's exception contract survives the boundary
  bool threw = false;
  try {
    std::vector<S> bad(q.begin(), q.end() - 1);
    gpu::fmm_apply(gplan, bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) std::printf("%-28s size mismatch did not throw std::invalid_argument FAIL\n", name);
  // the whole pipeline on the GPU from the points alone: same tree (pair counts
  // identical), own skeletons (agreement within the ID tolerance)
  ApplyStats s_pipe;
  gpu::GpuPlan<K> gpipe = gpu::GpuPlan<K>::from_points(kern, pts, leaf, tol);
  const std::vector<S> u_pipe = gpu::fmm_apply(gpipe, q, &s_pipe);
  const double err_pipe = rel_l2(u_pipe, u_cpu);
  const bool pipe_ok = err_pipe <= 10 * tol && s_pipe.n_ifo_pairs == s_cpu.n_ifo_pairs &&
                       s_pipe.n_ifs_pairs == s_cpu.n_ifs_pairs &&
                       s_pipe.n_tfo_pairs == s_cpu.n_tfo_pairs &&
                       s_pipe.n_level1_pairs == s_cpu.n_level1_pairs;
  std::printf("%-28s GPU pipeline rel_l2 vs CPU %.3e (bar %.0e) %s\n", name, err_pipe, 10 * tol,
              pipe_ok ? "OK" : "FAIL");
  return ok && threw && pipe_ok && multi_ok ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    g_devices.clear();
    for (const char* c = argv[1]; *c;) {
      g_devices.push_back(std::atoi(c));
      while (*c && *c != ',') ++c;
      if (*c == ',') ++c;
    }
  }
  int fails = 0;
  fails += run("laplace3d cube", Laplace3d{}, Distribution::cube, 20000, 64, 1e-6);
  fails += run("laplace3d sphere tol1e-8", Laplace3d{}, Distribution::sphere, 20000, 40, 1e-8);
  fails += run("laplace2d square", Laplace2d{}, Distribution::square, 20000, 64, 1e-6);
  fails += run("laplace2d annulus", Laplace2d{}, Distribution::annulus, 8000, 30, 1e-6);
  fails += run("helmholtz3d cube k=10", Helmholtz3d{10.0}, Distribution::cube, 8000, 64, 1e-6);
  fails += run("laplace3d depth0 fallback", Laplace3d{}, Distribution::cube, 50, 100, 1e-6);
  std::printf("%s\n", fails ? "DROPIN PARITY FAIL" : "DROPIN PARITY OK");
  return fails ? 1 : 0;
}
