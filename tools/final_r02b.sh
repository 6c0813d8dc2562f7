#!/bin/bash
# Round-2 closing measurements on the final sources (GPU box, repo root):
# launch list + ncu --set full captures of K2 (headline, sphere, 2-D) and of
# the two-pass K4, each profiled command first run plain; then the GPU test
# suite, smoke, the headline bench line with the CPU reference legs, every
# BASELINE config, config 5 on one GPU and the 1-rank NCCL path.
set -u
out=gpurun_out/final2
mkdir -p $out/configs
H="python bench.py --steps 2 --warmup 3 --cpu off --check-targets 10"
$H > $out/plain_h.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_1e7.csv $H > $out/ncu_launches.log 2>&1
K="python bench.py --steps 1 --warmup 3 --cpu off --check-targets 10"
$K > $out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_translate -s 3 -c 1 \
    -o $out/k2_full $K > $out/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_ -s 6 -c 2 \
    -o $out/k4_full $K > $out/ncu_k4.log 2>&1
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
for c in c1 c2 c3a c3b c4; do
  python bench.py --config $c --steps 10 --warmup 3 > $out/configs/bench_$c.json 2> $out/configs/bench_$c.err
done
python bench.py --config c5 --steps 3 --warmup 3 --cpu off > $out/configs/bench_c5_1gpu_1e8.json 2> $out/configs/bench_c5.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --force-sharded --steps 5 --warmup 3 > $out/bench_sharded_1rank_nccl.json 2> $out/sharded.err
ls -la $out $out/configs
