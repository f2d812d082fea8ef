# L=100: 64 + 40 fields (full chunk unrolled, remainder runtime loop) vs an even 56 + 56 split with a
# 7-batch unrolled copy (PI2_TC_EVEN_SPLIT + PI2_TC_UNROLL56)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "" "-DPI2_TC_EVEN_SPLIT -DPI2_TC_UNROLL56" "" "-DPI2_TC_EVEN_SPLIT -DPI2_TC_UNROLL56"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 110; do timeout 60 /tmp/tct 3276800 $L | grep -E "rows|tensor-core"; done
done
