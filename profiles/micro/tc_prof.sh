#!/bin/bash
# lwpr_tc_kernel vs the CUDA-core kernel (C2 rows, L = 100 and 200), then phase clocks (PI2_TC_PROF)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in "4 64" "3 64"; do
  set -- $v
  $B -DPI2_TC_CTAS=$1 -DPI2_TC_CHUNK=$2 -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  timeout 60 /tmp/tct 3276800 100
  timeout 60 /tmp/tct 3276800 200 | grep -E "us|dmean|fit"
  $B -DPI2_TC_PROF -DPI2_TC_CTAS=$1 -DPI2_TC_CHUNK=$2 -o /tmp/tctp profiles/micro/lwpr_tc_test.cu || continue
  timeout 60 /tmp/tctp 3276800 100 | grep clocks
done
