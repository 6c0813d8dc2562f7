#!/bin/bash
# Round-2 final numbers on the GPU box (repo root): GPU test suite, smoke, the
# headline bench line (with the CPU reference legs) and every BASELINE config.
set -u
out=gpurun_out/r02
mkdir -p $out/configs
timeout 1800 python -m pytest tests -m gpu -q > $out/gputest.log 2>&1; echo "exit $?" >> $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "exit $?" >> $out/smoke.log
python bench.py > $out/bench_headline_1e7.json 2> $out/bench_headline_1e7.err
for c in c1 c2 c3a c3b c4; do
  python bench.py --config $c --steps 10 --warmup 3 > $out/configs/bench_$c.json 2> $out/configs/bench_$c.err
done
python bench.py --config c5 --steps 3 --warmup 3 --cpu off > $out/configs/bench_c5_1gpu_1e8.json 2> $out/configs/bench_c5.err
ls -la $out $out/configs
