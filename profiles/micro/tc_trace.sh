# phase trace (PI2_TC_TRACE) of the tensor-core LWPR kernels on SM 0: per SM sub-partition, the time
# share with n warps in the exp phase, phase totals, and a timeline window
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_TRACE -o /tmp/tctr profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for v in 1; do echo "== TC3=$v L=100"; TC3=$v timeout 60 /tmp/tctr 3276800 100 | grep -E "SMSP|  w|tensor-core"; done
