#!/bin/bash
# Round evidence on one B200: bench lines (ours, reference arm), ncu launch list and one
# `ncu --set full` capture of a C2 control-step iteration.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1 || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1 || exit 1
python profiles/profile_step.py --iters 2 > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python profiles/profile_step.py --iters 2 > gpurun_out/ncu_launch.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -c 6 -f -o gpurun_out/prof_final \
  python profiles/profile_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1 || exit 1
echo done
