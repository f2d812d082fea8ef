# attitude_kernel: noise look-ahead TB and outer-loop unroll; C2 / C4 device ms per step
cd $GRAFT_REPO_ROOT
for f in "-DPI2_ATT_TB=4 -DPI2_ATT_UNROLL=1" "-DPI2_ATT_TB=8 -DPI2_ATT_UNROLL=1" "-DPI2_ATT_TB=2 -DPI2_ATT_UNROLL=1" "-DPI2_ATT_TB=4 -DPI2_ATT_UNROLL=2" "-DPI2_ATT_TB=4 -DPI2_ATT_UNROLL=1" "-DPI2_ATT_TB=8 -DPI2_ATT_UNROLL=1"; do
  PI2_NVCC_EXTRA="$f" python -m paper_1503_00330_b200._build --force > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  for c in C2 C4; do
    echo "$f $c $(python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --closed-loop-steps 0 | tail -1 | grep -o '"ms_per_step": [0-9.]*') att $(python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --closed-loop-steps 0 | tail -1 | grep -o '"attitude": [0-9.]*')"
  done
done
python -m paper_1503_00330_b200._build --force > /dev/null 2>&1
