# remainder chunk's exp loop unrolled at a compile-time batch count (-DPI2_TC_REMB=5: L=100's 40-field
# remainder) vs the runtime loop
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -o /tmp/tcr0 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_REMB=5 -o /tmp/tcr5 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_REMB=1 -o /tmp/tcr1 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for r in 1 2; do for v in 0 5; do echo "== REMB=$v L=100 round $r"; timeout 60 /tmp/tcr$v 3276800 100 | grep -E "tensor-core|hash"; done; done
for r in 1 2; do for v in 0 1; do echo "== REMB=$v L=200 round $r"; timeout 60 /tmp/tcr$v 3276800 200 | grep -E "tensor-core|hash"; done; done
