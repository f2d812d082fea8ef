# exp loop: full chunks unrolled + runtime remainder loop (PI2_TC_UNROLL=1) vs one loop unrolled
# to 8 batches with a uniform guard per pair for every chunk (PI2_TC_UNROLL=3)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "-DPI2_TC_UNROLL=1" "-DPI2_TC_UNROLL=3" "-DPI2_TC_UNROLL=1" "-DPI2_TC_UNROLL=3"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 200 64 130 48; do timeout 60 /tmp/tct 3276800 $L | grep -E "rows|us|dmean"; done
done
