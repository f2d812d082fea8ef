# warp-specialised TMEM multi-buffered LWPR kernel (lwpr_tcws_kernel, WS=1) vs lwpr_tc_kernel (WS=0), at
# 64-field chunks (2 buffers) and 32-field chunks (4 buffers): time and output bit hashes
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for c in 64 32; do $B -DPI2_TC_CHUNK=$c -o /tmp/tcws$c profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
$B -DPI2_TC_CHUNK=32 -DPI2_TC_TRACE -o /tmp/tcwst profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 1000; do
  for cv in "64 0" "64 1" "32 0" "32 1"; do set -- $cv; echo "== chunk $1 WS=$2 L=$L"; WS=$2 timeout 60 /tmp/tcws$1 3276800 $L | grep -E "tensor-core|hash|W "; done
done
for R in 51200 129; do for cv in "64 0" "32 1"; do set -- $cv; echo "== chunk $1 WS=$2 rows=$R L=100"; WS=$2 timeout 60 /tmp/tcws$1 $R 100 | grep -E "tensor-core"; done; done
echo "== trace chunk 32 WS=1 L=100"; WS=1 timeout 60 /tmp/tcwst 3276800 100 | grep -E "SMSP"
