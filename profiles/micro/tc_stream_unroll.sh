# streamed weights (L=1000, PI2_LWPR_TC_STREAM=1): pipelined runtime loop (PI2_TC_LDPIPE=1, default)
# vs the unrolled full-chunk loop (PI2_TC_LDPIPE=0 -> the resident path's loop)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "-DPI2_TC_LDPIPE=1" "-DPI2_TC_LDPIPE=0" "-DPI2_TC_LDPIPE=1" "-DPI2_TC_LDPIPE=0"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 1000 300; do PI2_LWPR_TC_STREAM=1 timeout 60 /tmp/tct 3276800 $L | grep -E "rows|tensor-core"; done
done
