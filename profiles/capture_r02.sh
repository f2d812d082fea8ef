#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun); outputs under ${OUT:-gpurun_out}/r02/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}/r02"
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err || exit 1
python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference_arm.json 2> $OUT/bench_ref.err || exit 1
for c in C1 C3 C5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-north-star > $OUT/bench_$c.json 2> $OUT/bench_$c.err || exit 1
done
python profiles/noise_stream.py > $OUT/noise_stream.json 2>&1 || exit 1
python profiles/k_sweep.py > $OUT/c5_k_sweep.txt 2>&1 || exit 1
# launch lists (cold, serialised): the bench command itself, and C2 / C4 steps (also without the
# inter-kernel cache flush, for the step's real DRAM traffic)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --closed-loop-steps 0 > $OUT/ncu_launch_bench.log 2>&1 || exit 1
for c in C2 C4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_$c.csv python profiles/profile_step.py --config $c --iters 2 > $OUT/ncu_launch_$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
    --csv --log-file $OUT/launches_${c}_nocc.csv python profiles/profile_step.py --config $c --iters 3 > $OUT/ncu_launch_${c}_nocc.log 2>&1 || exit 1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"attitude|rollout" --log-file $OUT/noise_stream_ncu.csv python profiles/noise_stream.py --reps 1 \
  > $OUT/ncu_noise.log 2>&1 || exit 1
# one full capture of the dominant kernel (C2 variance path, C4 mean-only path)
ncu --set full --clock-control none --import-source on -k regex:lwpr_tc -c 1 -f -o $OUT/lwpr_c2 \
  python profiles/profile_step.py --iters 1 > $OUT/ncu_full_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:lwpr_tc -c 1 -f -o $OUT/lwpr_c4 \
  python profiles/profile_step.py --config C4 --iters 1 > $OUT/ncu_full_c4.log 2>&1 || exit 1
echo done
