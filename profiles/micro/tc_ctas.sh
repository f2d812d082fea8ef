#!/bin/bash
# co-resident CTAs per SM x field chunk (TMEM = 2 x chunk columns per CTA)
cd $GRAFT_REPO_ROOT
for v in "4 64" "6 32" "8 32" "5 32"; do
  set -- $v
  echo "== CTAS $1 CHUNK $2"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc \
    -DPI2_TC_CTAS=$1 -DPI2_TC_CHUNK=$2 -Xptxas -v -o /tmp/tct profiles/micro/lwpr_tc_test.cu 2>&1 | grep -A2 "lwpr_tc_kernelILb1ELb0" | grep -E "spill|Used" | tr '\n' ' '; echo
  for L in 100 200; do timeout 60 /tmp/tct 3276800 $L | grep -E "W |cuda-core|mean-only|fit"; done
done
