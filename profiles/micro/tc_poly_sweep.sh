# re-tune of the FMA-pipe 2^x share after the two-MMA packing and the remainder unroll:
# POLY_VAR / POLY_VAR_B (variance loop), POLY_MEAN / POLY_MEAN_B (mean-only), field pairs of 4 per batch
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for cfg in "0 1 1 1" "0 0 1 1" "0 2 1 1" "1 1 1 1" "1 0 1 1" "0 1 1 0" "0 1 2 1" "0 1 1 2" "0 1 2 2" "0 1 0 1"; do
  set -- $cfg
  $B -DPI2_TC_POLY_VAR=$1 -DPI2_TC_POLY_VAR_B=$2 -DPI2_TC_POLY_MEAN=$3 -DPI2_TC_POLY_MEAN_B=$4 -o /tmp/tps profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
  for L in 100 200; do echo "== VAR $1/$2 MEAN $3/$4 L=$L"; timeout 60 /tmp/tps 3276800 $L | grep -E "tensor-core"; done
done
