# remainder chunk's exp loop: bounded-unrolled with a runtime count (PI2_TC_REM_UNROLL=1) vs the runtime loop (0)
# vs a compile-time count (-DPI2_TC_REMB=5, L=100 only)
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_REM_UNROLL=0 -o /tmp/tcu0 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_REM_UNROLL=1 -o /tmp/tcu1 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_REM_UNROLL=0 -DPI2_TC_REMB=5 -o /tmp/tcu5 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 130 1000 48; do for r in 1 2; do for v in 0 1 5; do
  [ $v = 5 ] && [ $L != 100 ] && continue
  echo "== variant $v L=$L round $r"; timeout 60 /tmp/tcu$v 3276800 $L | grep -E "tensor-core|hash"; done; done; done
