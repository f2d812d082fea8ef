# rollout_group_kernel t-loop unroll 4 (default) vs 8 (C2 device ms per step)
cd $GRAFT_REPO_ROOT
for f in "-DPI2_ROLL_UNROLL=4" "-DPI2_ROLL_UNROLL=8" "-DPI2_ROLL_UNROLL=4" "-DPI2_ROLL_UNROLL=8"; do
  PI2_NVCC_EXTRA="$f" python -m paper_1503_00330_b200._build --force > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  echo "$f C2 $(python bench.py --config C2 --steps 50 --warmup 3 --no-cpu-baseline --closed-loop-steps 0 | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done
python -m paper_1503_00330_b200._build --force > /dev/null 2>&1
