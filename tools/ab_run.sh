#!/bin/bash
# A/B of library variants (tools/build_variant.sh) on one bench command:
#   VARIANTS="base v1 v2" bash tools/ab_run.sh TAG <bench args...>
# prints value, step ms, K2 ms and the accuracy check per variant.
tag=$1; shift
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset SFMM_LIB_DIR; else export SFMM_LIB_DIR=build/$v; fi
  python bench.py "$@" > gpurun_out/ab_${tag}_$v.json 2> gpurun_out/ab_${tag}_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${tag}_$v.json'))
print('$tag', '$v', round(d['value'],2), round(d['ms_per_step'],3), round(d['phase_ms']['translate'],3), d.get('relerr_vs_direct'))"
done
