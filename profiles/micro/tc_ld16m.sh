# mean-only kernel: 16-column logits + two 8-column y' loads (PI2_TC_LD16M; record, code reverted)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "-DPI2_TC_LD16M=0" "-DPI2_TC_LD16M=1" "-DPI2_TC_LD16M=0" "-DPI2_TC_LD16M=1"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 200 64; do timeout 60 /tmp/tct 3276800 $L | grep -E "rows|tensor-core"; done
done
