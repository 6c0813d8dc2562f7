#!/bin/bash
# A/B of the 512-entry log table (SFMM_LOG_BITS=9, build/log9) on the 2-D configs.
set -u
out=gpurun_out/ablog9; mkdir -p $out
for v in base log9 base log9; do
  if [ $v = base ]; then unset SFMM_LIB_DIR; else export SFMM_LIB_DIR=build/log9; fi
  python bench.py --config c1 --steps 50 --warmup 5 --cpu-reps 1 --cpu-native 0 > $out/c1_$v.json 2> $out/c1_$v.err
  python -c "
import json; d=json.load(open('$out/c1_$v.json'))
print('c1', '$v', round(d['value'],2), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()}, d.get('relerr_vs_cpu_ref'), d.get('max_relerr_vs_cpu_ref'))"
done
for v in base log9; do
  if [ $v = base ]; then unset SFMM_LIB_DIR; else export SFMM_LIB_DIR=build/log9; fi
  python bench.py --kernel laplace2d --dist square --points 4e6 --leaf 64 --steps 10 --warmup 3 --cpu off > $out/sq4e6_$v.json 2> $out/sq4e6_$v.err
  python -c "
import json; d=json.load(open('$out/sq4e6_$v.json'))
print('square 4e6', '$v', round(d['value'],2), round(d['ms_per_step'],4), round(d['phase_ms']['translate'],4), d.get('relerr_vs_direct'))"
done
SFMM_LIB_DIR=build/log9 timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_apply_gpu.py -m gpu -q -x -k "log or golden or laplace2d or annulus or square" > $out/tests_log9.log 2>&1; echo "exit $?" >> $out/tests_log9.log
tail -2 $out/tests_log9.log
