set -e
bash tools/cmp_variants.sh "c4 c3 c5" "base"
for c in c4 c3; do
ncu --set full --clock-control none --import-source on -k regex:nlm_pass3 -c 2 -f -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$c.log 2>&1 || tail -5 gpurun_out/ncu_$c.log
done
ls -la gpurun_out/*.ncu-rep
