for v in ${VARIANTS:-base u2 u2b3 r4b3 r3b3 r4b4}; do
  if [ $v = base ]; then unset SFMM_LIB_DIR; else export SFMM_LIB_DIR=build/$v; fi
  python bench.py --kernel helmholtz3d --points 2e6 --steps 5 --warmup 3 --cpu off --check-targets 200 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],2), round(d['phase_ms']['translate'],2), d.get('relerr_vs_direct'))"
done
