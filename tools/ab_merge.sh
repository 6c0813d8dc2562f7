#!/bin/bash
# A/B of merged multi-tile K2 tasks (SFMM_MERGE_TILES) and the low-memory layout choice.
set -u
out=gpurun_out/abmerge2; mkdir -p $out
run() {  # tag env args...
  tag=$1; shift; envs=$1; shift
  env $envs timeout 1500 python bench.py "$@" --cpu off > $out/$tag.json 2> $out/$tag.err
  python -c "
import json; d=json.load(open('$out/$tag.json'))
print('$tag', round(d['value'],2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, d.get('relerr_vs_direct'), d.get('sym_staging'), d.get('resident_plan_gb'))" 2>&1 | tail -1
}
run h_def X=1 --steps 10 --warmup 3
run h_m1 SFMM_MERGE_TILES=1 --steps 10 --warmup 3
run h_chain SFMM_SYM_CHAIN=1 --steps 5 --warmup 3
run c2_def X=1 --config c2 --steps 10 --warmup 3
run c3a_def X=1 --config c3a --steps 5 --warmup 3
run c5_def X=1 --config c5 --steps 3 --warmup 3
