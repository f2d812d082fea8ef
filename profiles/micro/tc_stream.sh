#!/bin/bash
# streamed-W tensor-core LWPR (large L) vs the CUDA-core kernel; L=100 also forced-streamed
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc -o /tmp/tct profiles/micro/lwpr_tc_test.cu || exit 1
timeout 60 /tmp/tct 3276800 100
STREAM=1 timeout 60 /tmp/tct 3276800 100
timeout 120 /tmp/tct 1310720 500
timeout 120 /tmp/tct 655360 1000
