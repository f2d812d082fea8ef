# phase clocks (PI2_TC_PROF) of the tensor-core LWPR kernel after the exp-loop unroll, L = 100 and 200
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_PROF -o /tmp/tctp profiles/micro/lwpr_tc_test.cu || exit 1
for L in 100 200 64; do echo "L=$L"; timeout 60 /tmp/tctp 3276800 $L | grep -E "clocks|tensor-core"; done
