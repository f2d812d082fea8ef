#!/bin/bash
# re-tune of the FMA-pipe 2^x share after the exp loop was unrolled (PI2_TC_UNROLL=1):
# field pairs (of 4) of the first / second 8-field batch, variance and mean-only loops
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in "0 1 1 1" "0 0 1 1" "1 1 1 1" "0 1 1 2" "1 1 2 2" "0 2 0 1" "0 1 0 0"; do
  set -- $v
  echo "== POLY_VAR $1/$2 POLY_MEAN $3/$4"
  $B -DPI2_TC_POLY_VAR=$1 -DPI2_TC_POLY_VAR_B=$2 -DPI2_TC_POLY_MEAN=$3 -DPI2_TC_POLY_MEAN_B=$4 -o /tmp/tct profiles/micro/lwpr_tc_test.cu || continue
  for L in 100 200; do timeout 60 /tmp/tct 3276800 $L | grep -E "tensor-core"; done
done
