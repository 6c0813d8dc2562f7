#!/bin/bash
# Builds libsfmm_gpu.so with extra -D flags into build/<name>/ (A/B runs via
# SFMM_LIB_DIR=build/<name>; the host library is copied alongside).
set -e
name=$1; shift
out=build/$name
mkdir -p $out/obj
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fopenmp -Iinclude -Ipaper_2310_16668_b200/csrc --expt-relaxed-constexpr $*"
objs=""
for f in kernels_translate kernels_tree kernels_multi skel_gpu tree_gpu sfmm_gpu sfmm_multi; do
  /usr/local/cuda/bin/nvcc $FL -c paper_2310_16668_b200/csrc/$f.cu -o $out/obj/$f.o &
  objs="$objs $out/obj/$f.o"
done
g++ -std=c++17 -O2 -fopenmp -fPIC -Iinclude -Ipaper_2310_16668_b200/csrc -I/usr/local/cuda/include $* \
    -c paper_2310_16668_b200/csrc/plan_build.cpp -o $out/obj/plan_build.o &
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -o $out/libsfmm_gpu.so $objs $out/obj/plan_build.o -lcudart_static -lgomp -lpthread -ldl -lrt
cp paper_2310_16668_b200/lib/libsfmm_host.so paper_2310_16668_b200/lib/libsfmm_probe.so $out/
echo built $out
