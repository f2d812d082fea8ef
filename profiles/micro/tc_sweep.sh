#!/bin/bash
# build + run lwpr_tc_test variants: WG PIPE ACC2 CTAS CHUNK
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "1 0 0 4 64" "1 1 0 4 64" "1 0 1 4 64" "1 1 1 4 64" "2 0 1 3 64" "2 1 1 3 64" "2 1 1 4 64" "2 1 1 2 64" "1 1 1 3 64"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc \
    -DPI2_TC_WG=$1 -DPI2_TC_PIPE=$2 -DPI2_TC_ACC2=$3 -DPI2_TC_CTAS=$4 -DPI2_TC_CHUNK=$5 -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  timeout 60 /tmp/tct 3276800 100
  timeout 60 /tmp/tct 3276800 200 | tail -3
done
