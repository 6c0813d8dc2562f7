#!/bin/bash
# Closing re-capture after the 512-entry log table (fastmath.cuh changed, so the
# K2 source hash did): ncu --set full of K2 at the headline, config 3a and
# config 1, the GPU test suite, smoke, the headline line and config 1.
set -u
out=gpurun_out/final3
mkdir -p $out/configs
K="python bench.py --steps 1 --warmup 3 --cpu off --check-targets 10"
$K > $out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_full $K > $out/ncu_k2.log 2>&1
S="python bench.py --config c3a --steps 1 --warmup 2 --cpu off --check-targets 10"
$S > $out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 2 -c 1 \
    -o $out/k2_c3a $S > $out/ncu_c3a.log 2>&1
C="python bench.py --config c1 --steps 1 --warmup 3 --cpu off --graphs off --check-targets 10"
$C > $out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_c1 $C > $out/ncu_c1.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $out/gputest.log 2>&1; echo "exit $?" >> $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "exit $?" >> $out/smoke.log
python bench.py > $out/bench_headline_1e7.json 2> $out/bench_headline_1e7.err
python bench.py --config c1 --steps 10 --warmup 3 > $out/configs/bench_c1.json 2> $out/configs/bench_c1.err
ls -la $out $out/configs
