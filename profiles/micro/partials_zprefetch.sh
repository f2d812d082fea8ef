# partials_kernel: stored normals loaded in the min pass (PI2_PARTIALS_ZPREFETCH=1) or after each exp (0)
cd $GRAFT_REPO_ROOT
for f in "-DPI2_PARTIALS_ZPREFETCH=0" "-DPI2_PARTIALS_ZPREFETCH=1" "-DPI2_PARTIALS_ZPREFETCH=0" "-DPI2_PARTIALS_ZPREFETCH=1"; do
  PI2_NVCC_EXTRA="$f" python -m paper_1503_00330_b200._build --force > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  for c in C2 C4; do
    echo "$f $c $(python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --closed-loop-steps 0 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"partials": [0-9.]*' | tr '\n' ' ')"
  done
done
python -m paper_1503_00330_b200._build --force > /dev/null 2>&1
