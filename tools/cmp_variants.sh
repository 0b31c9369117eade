# usage: bash tools/cmp_variants.sh "c4 c3 c5" "base B BC ..." [steps]  (variants under lib/var_<tag>)
# Prints value, row/col pass ms and frac per (config, variant); numbers from bench.py.
CFGS=${1:-"c4 c3 c5"}; VARS=${2:-"base"}; STEPS=${3:-10}
mkdir -p gpurun_out
for c in $CFGS; do
  for v in $VARS; do
    if [ $v = base ]; then L=""; else L="PLGPU_LIB=paper_1407_2343_b200/lib/var_$v/libplgpu.so"; fi
    env $L python bench.py --config $c --steps $STEPS --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cmp_${c}_$v.log 2>&1
    python -c "
import json,sys
l=json.loads([x for x in open('gpurun_out/cmp_${c}_$v.log') if x.startswith('{')][-1])
r=l['roofline'];print('$c','$v',round(l['value']),round(r['row_pass_ms'],4),round(r['col_pass_ms'],4),round(r['frac'],4), l['e2e'].get('matches_device_result'))" || tail -3 gpurun_out/cmp_${c}_$v.log
  done
done
