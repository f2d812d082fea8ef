# lwpr_tc3_kernel SPLIT=1 (2 CTAs/SM x 4 warps, TMEM double-buffered 64-field items) vs lwpr_tc_kernel
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -o /tmp/tc4h profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_TRACE -o /tmp/tc4t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 1000; do
  for v in 0 1; do echo "== TC3=$v L=$L"; TC3=$v timeout 60 /tmp/tc4h 3276800 $L | grep -E "tensor-core|max"; done
done
echo "== trace TC3=1 L=100"; TC3=1 timeout 60 /tmp/tc4t 3276800 100 | grep -E "SMSP"
