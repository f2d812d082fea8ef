#!/bin/bash
# Round evidence on one B200: bench lines (ours, reference arm), ncu launch list and one
# `ncu --set full` capture of a C2 control-step iteration.  Outputs under ${OUT:-gpurun_out}/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}"
mkdir -p "$OUT"
python bench.py > $OUT/bench_default.log 2>&1 || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1 || exit 1
python profiles/profile_step.py --iters 2 > $OUT/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python profiles/profile_step.py --iters 2 > $OUT/ncu_launch.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --closed-loop-steps 0 > $OUT/ncu_launch_bench.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -c 6 -f -o $OUT/prof_final \
  python profiles/profile_step.py --iters 1 > $OUT/ncu_full.log 2>&1 || exit 1
echo done
