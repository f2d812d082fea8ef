# software-pipelined TMEM loads in the exp loop (PI2_TC_LDPIPE) vs load-2-wait-compute-2
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for d in "-DPI2_TC_LDPIPE=0" "-DPI2_TC_LDPIPE=1" "-DPI2_TC_LDPIPE=0" "-DPI2_TC_LDPIPE=1"; do
  echo "== $d"
  $B $d -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 200; do timeout 60 /tmp/tct 3276800 $L | grep -E "rows|us|dmean"; done
  PI2_LWPR_TC_STREAM=1 timeout 60 /tmp/tct 3276800 1000 | grep -E "rows|us|dmean"
done
