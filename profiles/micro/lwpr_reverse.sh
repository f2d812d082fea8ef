# DRAM bytes per kernel of a C2 / C4 step WITHOUT ncu's cache flush between kernels (--cache-control none),
# LWPR tiles in reverse row order (PI2_TC_REVERSE=1, default) vs forward (0); stage times with each build
cd $GRAFT_REPO_ROOT
for v in 1 0; do
  PI2_NVCC_EXTRA="-DPI2_TC_REVERSE=$v" python -c "from paper_1503_00330_b200 import _build; _build.build(force=True)" || exit 1
  for c in C2 C4; do
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
      --csv --log-file gpurun_out/rev${v}_nocc_$c.csv python profiles/profile_step.py --config $c --iters 3 > /dev/null 2>&1
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/rev${v}_flush_$c.csv python profiles/profile_step.py --config $c --iters 3 > /dev/null 2>&1
  done
  echo "REVERSE=$v"; python profiles/micro/roll_variant.py --config C2 --env PI2_NONE_A 2>&1 | tail -3 | head -1
  python profiles/micro/roll_variant.py --config C4 --env PI2_NONE_A 2>&1 | tail -3 | head -1
done
