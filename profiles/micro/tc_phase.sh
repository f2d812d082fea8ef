#!/bin/bash
# phase clocks of the current lwpr_tc_kernel (PI2_TC_PROF), variance path, L = 100 and 200
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc -DPI2_TC_PROF \
  -o /tmp/tctp profiles/micro/lwpr_tc_test.cu || exit 1
for L in 100 200; do timeout 60 /tmp/tctp 3276800 $L | grep -E "rows|clocks|cuda-core"; done
