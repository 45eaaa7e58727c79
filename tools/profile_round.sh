#!/bin/bash
# One GPU-box pass of the round's evidence: tests, bench line, ncu launch list,
# ncu --set full captures (each only after its command has run clean without ncu).
#   tools/profile_round.sh TAG      -> gpurun_out/TAG/*
tag=${1:-r02}
O=gpurun_out/$tag
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
if [ -z "$SKIP_TESTS" ]; then
  (time python -m pytest tests -m gpu -x -q --durations=10) > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
fi
python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
cap() {  # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  "$@" > $O/$name.plain.log 2>&1 || { echo "plain run failed: $name" >> $O/errors.txt; return; }
  $NCU -k regex:$rx --launch-skip $skip -c 1 -f -o $O/$name "$@" > $O/$name.ncu.log 2>&1
  if [ -f $O/$name.ncu-rep ]; then
    bash tools/ncu_summary.sh $O/$name.ncu-rep > $O/$name.txt 2>&1
    ncu -i $O/$name.ncu-rep --page source --csv --print-source=cuda,sass 2>/dev/null | gzip > $O/$name.source.csv.gz
    [ -n "$KEEP_REPS" ] || rm -f $O/$name.ncu-rep
  else
    echo "no report: $name" >> $O/errors.txt
  fi
}
cap ncu_bench_admm convex_kernel 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --only admm_l0.1
cap ncu_bench_fista convex_kernel 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --only fista_l0.1
cap ncu_sse_coeff sse_coeff_kernel 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --only fista_l100
cap ncu_gomp_warp27 gomp_warp_kernel 0 python tools/run_case.py --cube salinas --algo gomp --kappa 27 --pixels 40000 --reps 1
cap ncu_biht27 greedy_kernel 0 python tools/run_case.py --cube salinas --algo biht --kappa 27 --pixels 40000 --reps 1
cap ncu_cosamp27 greedy_kernel 0 python tools/run_case.py --cube salinas --algo cosamp --kappa 27 --pixels 40000 --reps 1
ls -la $O
