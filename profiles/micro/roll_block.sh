# threads per block of the attitude / rollout kernels (PI2_ROLL_BLOCK): C2 / C4 device ms per step
cd $GRAFT_REPO_ROOT
for f in "-DPI2_ROLL_BLOCK=128" "-DPI2_ROLL_BLOCK=64" "-DPI2_ROLL_BLOCK=256" "-DPI2_ROLL_BLOCK=128" "-DPI2_ROLL_BLOCK=64" "-DPI2_ROLL_BLOCK=256"; do
  PI2_NVCC_EXTRA="$f" python -m paper_1503_00330_b200._build --force > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  for c in C2 C4; do
    echo "$f $c $(python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --closed-loop-steps 0 | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  done
done
python -m paper_1503_00330_b200._build --force > /dev/null 2>&1
