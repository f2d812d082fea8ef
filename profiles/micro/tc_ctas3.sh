cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for n in 4 3; do $B -DPI2_TC_CTAS=$n -o /tmp/tcc$n profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
for L in 100 200; do for n in 4 3; do echo "== CTAS=$n L=$L"; timeout 60 /tmp/tcc$n 3276800 $L | grep -E "tensor-core"; done; done
