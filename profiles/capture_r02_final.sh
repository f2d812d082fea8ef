#!/bin/bash
# End-of-round-2 evidence on one B200 (run under gpurun); outputs under ${OUT:-gpurun_out}/r02f/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}/r02f"
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
timeout 1200 python -m pytest tests -m gpu -q > $OUT/gputest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
python bench.py > $OUT/bench.json 2> $OUT/bench.err || exit 1
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference_arm.json 2> $OUT/bench_ref.err || exit 1
# launch lists (cold, serialised): the bench command itself, and C2 / C4 steps with DRAM bytes
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --closed-loop-steps 0 --no-other-configs --no-north-star \
  > $OUT/ncu_launch_bench.log 2>&1 || exit 1
for c in C2 C4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_$c.csv python profiles/profile_step.py --config $c --iters 2 > $OUT/ncu_launch_$c.log 2>&1 || exit 1
done
# full captures: the dominant kernel at C2 (variance) and C4 (mean-only), partials at C4
ncu --set full --clock-control none --import-source on -k regex:lwpr_tc -c 1 -f -o $OUT/lwpr_c2 \
  python profiles/profile_step.py --iters 1 > $OUT/ncu_full_lwpr_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:lwpr_tc -c 1 -f -o $OUT/lwpr_c4 \
  python profiles/profile_step.py --config C4 --iters 1 > $OUT/ncu_full_lwpr_c4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:partials -c 1 -f -o $OUT/partials_c4 \
  python profiles/profile_step.py --config C4 --iters 1 > $OUT/ncu_full_partials_c4.log 2>&1 || exit 1
echo done
