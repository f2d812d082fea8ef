cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_CHUNK=${CHUNK:-32} -DPI2_TC_TRACE -o /tmp/tcwst profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
echo "== trace chunk ${CHUNK:-32} WS=1 L=100"; WS=1 timeout 60 /tmp/tcwst 3276800 100 | grep -E "SMSP|  w"
