# proxy fence only at a tile's first chunk (PI2_TC_FENCE_C0=1) vs every chunk (0): time and bit hashes
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in 0 1; do $B -DPI2_TC_FENCE_C0=$v -o /tmp/tcf$v profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
for L in 100 200 1000; do for r in 1 2; do for v in 0 1; do echo "== FENCE_C0=$v L=$L round $r"; timeout 60 /tmp/tcf$v 3276800 $L | grep -E "tensor-core|hash"; done; done; done
