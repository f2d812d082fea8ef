# remainder-chunk pairs with 16-column tcgen05.ld (PI2_TC_LD16R; record, code reverted)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "-DPI2_TC_LD16R=0" "-DPI2_TC_LD16R=1" "-DPI2_TC_LD16R=0" "-DPI2_TC_LD16R=1"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 110 130; do timeout 60 /tmp/tct 3276800 $L | grep -E "rows|tensor-core"; done
done
