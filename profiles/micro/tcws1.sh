# lwpr_tcws_kernel with ONE producer warp per CTA (4 CTAs/SM x (4 exp + 1 producer warps), 32-field chunks
# double-buffered in 128 TMEM columns) vs lwpr_tc_kernel at 64-field chunks
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_CHUNK=64 -DPI2_TCWS_P=4 -o /tmp/tcold profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_CHUNK=32 -DPI2_TCWS_P=1 -o /tmp/tcp1 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_CHUNK=32 -DPI2_TCWS_P=1 -DPI2_TC_TRACE -o /tmp/tcp1t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 1000; do
  echo "== old L=$L"; WS=0 timeout 60 /tmp/tcold 3276800 $L | grep -E "tensor-core|hash"
  echo "== P1 chunk 32 L=$L"; WS=1 timeout 60 /tmp/tcp1 3276800 $L | grep -E "tensor-core|hash|does not"
done
echo "== trace P1"; WS=1 timeout 60 /tmp/tcp1t 3276800 100 | grep -E "SMSP|  w"
