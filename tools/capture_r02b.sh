#!/bin/bash
# Round-2 final evidence on the GPU box (repo root): the headline launch list,
# full ncu captures of K2 (headline, config 3a sphere) and K2m (config 4).
# Every profiled command first runs plain (must exit 0), as the profiling
# recipe requires.
set -u
out=gpurun_out/cap2
mkdir -p $out
H="python bench.py --steps 2 --warmup 3 --cpu off --check-targets 10"
$H > $out/plain_h.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_1e7.csv $H > $out/ncu_launches.log 2>&1
K="python bench.py --steps 1 --warmup 3 --cpu off --check-targets 10"
$K > $out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_full $K > $out/ncu_k2.log 2>&1
S="python bench.py --config c3a --steps 1 --warmup 2 --cpu off --check-targets 10"
$S > $out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 2 -c 1 \
    -o $out/k2_c3a $S > $out/ncu_c3a.log 2>&1
M="python bench.py --config c4 --steps 1 --warmup 1 --cpu off --check-targets 10"
$M > $out/plain_m.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2m -s 2 -c 2 \
    -o $out/k2m_c4 $M > $out/ncu_k2m.log 2>&1
ls -la $out
