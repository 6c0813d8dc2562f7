#!/bin/bash
# A/B of the two-pass K4 (k4_fold + k4_gather) against the one-pass scatter.
set -u
out=gpurun_out/abk4; mkdir -p $out
for cfg in "" "--config c2" "--config c3a" "--kernel helmholtz3d --kappa 10 --points 2e6"; do
  tag=$(echo "h $cfg" | tr -d ' -.' )
  for g in 1 0; do
    SFMM_K4_GATHER=$g timeout 900 python bench.py $cfg --steps 10 --warmup 3 --cpu off > $out/${tag}_$g.json 2> $out/${tag}_$g.err
    python -c "
import json; d=json.load(open('$out/${tag}_$g.json'))
print('$tag', 'k4gather=$g', round(d['value'],2), round(d['ms_per_step'],3), {k: round(v,4) for k,v in d['phase_ms'].items()}, d.get('relerr_vs_direct'), d.get('e2e',{}).get('value'))" 2>&1 | tail -1
  done
done
