#!/bin/bash
# Re-measures every committed number (run on the GPU box from the repo root):
#   bench lines for the headline and each BASELINE config, the ncu launch list of
#   the headline bench command and one full ncu capture of the translation kernel.
set -u
out=gpurun_out/refresh
mkdir -p $out
python bench.py --steps 10 --warmup 3 > $out/bench_1e7.json 2> $out/bench_1e7.err
for c in c1 c2 c3a c3b c4; do
  python bench.py --config $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
# launch list (per-launch device times, serialised, cold cache)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_1e7.csv python bench.py --steps 2 --warmup 3 --cpu off \
    > $out/ncu_launches.log 2>&1
# one full capture of K2 at the headline size (first launch after warm-up)
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_full python bench.py --steps 1 --warmup 3 --cpu off > $out/ncu_k2.log 2>&1
# multi-RHS (config 4) translation kernel
ncu --set full --clock-control none --import-source on -k regex:k2m -s 1 -c 1 \
    -o $out/k2m_full python bench.py --config c4 --steps 1 --warmup 1 --cpu off \
    > $out/ncu_k2m.log 2>&1
# the adaptive sphere (config 3a): K2 capture for the instruction-fetch / task-order story
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 2 -c 1 \
    -o $out/k2_c3a python bench.py --config c3a --steps 1 --warmup 2 --cpu off > $out/ncu_k2_c3a.log 2>&1
# single-RHS Helmholtz (the reference's call shape): bench line + complex K2 capture
python bench.py --kernel helmholtz3d --points 4e6 --steps 5 --warmup 3 --cpu off \
    > $out/bench_h3d_4e6_1rhs.json 2> $out/bench_h3d_4e6_1rhs.err
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_h3d python bench.py --kernel helmholtz3d --points 2e6 --steps 1 --warmup 3 \
    --cpu off --check-targets 0 > $out/ncu_k2_h3d.log 2>&1
ls -la $out
