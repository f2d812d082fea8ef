# column-split double-buffered LWPR kernel (lwpr_tc3_kernel, TC3=1) vs lwpr_tc_kernel (TC3=0)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -o /tmp/tc3h profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC3_SPLIT=2 -o /tmp/tc3s profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_TRACE -o /tmp/tc3t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 130 1000 48; do
  for v in 0 1; do echo "== TC3=$v L=$L"; TC3=$v timeout 60 /tmp/tc3h 3276800 $L | grep -E "tensor-core|max|W |first"; done
done
echo "== trace TC3=1 L=100"; TC3=1 timeout 60 /tmp/tc3t 3276800 100 | grep -E "SMSP"
echo "== small (C1-like rows)"; for v in 0 1; do TC3=$v timeout 60 /tmp/tc3h 51200 100 | grep -E "tensor-core|max"; done
echo "== ragged rows"; for v in 0 1; do TC3=$v timeout 60 /tmp/tc3h 1000003 100 | grep -E "tensor-core|max"; done
