# 3xTF32 as two MMAs per chunk (PI2_TC_PACK2=1) vs three (0): time and accuracy against the CUDA-core kernel
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in 0 1; do $B -DPI2_TC_PACK2=$v -o /tmp/tcpk$v profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
$B -DPI2_TC_PACK2=1 -DPI2_TC_TRACE -o /tmp/tcpk1t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 1000; do for r in 1 2; do for v in 0 1; do echo "== PACK2=$v L=$L round $r"; timeout 60 /tmp/tcpk$v 3276800 $L | grep -E "tensor-core|max"; done; done; done
for v in 0 1; do echo "== PACK2=$v rows=51200"; timeout 60 /tmp/tcpk$v 51200 100 | grep -E "tensor-core"; done
echo "== trace PACK2=1 L=100"; timeout 60 /tmp/tcpk1t 3276800 100 | grep SMSP
