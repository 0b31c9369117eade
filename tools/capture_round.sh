# Round-end evidence capture on the GPU box: bench lines, launch list, ncu summaries.
# usage: [NCU_CFGS="c4 c3"] [SKIP_BENCH=1] bash tools/capture_round.sh <tag>
# (gpurun copies back at most 64 MiB: one c5 ncu report is ~39 MB, capture it alone)
set -u
T=${1:-r01}
O=gpurun_out/$T
mkdir -p $O
if [ -z "${SKIP_BENCH:-}" ]; then
python bench.py > $O/bench_c4.log 2>&1; tail -c 400 $O/bench_c4.log
for c in c3 c5 c2 c1; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.log 2>&1
done
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launches.log 2>&1
fi
for c in ${NCU_CFGS:-c4 c3}; do
  ncu --set full --clock-control none --import-source on -k regex:nlm_pass3 -c 2 -f -o $O/prof_$c \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_$c.log 2>&1
done
ls -la $O
