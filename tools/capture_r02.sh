#!/bin/bash
# Round-2 evidence on the GPU box (repo root): the headline launch list and
# full ncu captures of the translation kernels.  Every profiled command first
# runs plain (must exit 0), as the profiling recipe requires.
set -u
out=gpurun_out/cap
mkdir -p $out
H="python bench.py --steps 2 --warmup 3 --cpu off --check-targets 10"
$H > $out/plain_h.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_1e7.csv $H > $out/ncu_launches.log 2>&1
K="python bench.py --steps 1 --warmup 3 --cpu off --check-targets 10"
$K > $out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_full $K > $out/ncu_k2.log 2>&1
M="python bench.py --config c4 --points 1e6 --steps 1 --warmup 1 --cpu off --check-targets 10"
$M > $out/plain_m.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2m -s 2 -c 2 \
    -o $out/k2m_1e6 $M > $out/ncu_k2m.log 2>&1
C="python bench.py --config c1 --steps 1 --warmup 3 --cpu off --graphs off --check-targets 10"
$C > $out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_c1 $C > $out/ncu_c1.log 2>&1
ls -la $out
