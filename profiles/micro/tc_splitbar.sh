# split-barrier LWPR schedule (PI2_TC_SPLITBAR=1) vs the CTA-barrier schedule (0): time and output bit hashes
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in 0 1; do $B -DPI2_TC_SPLITBAR=$v -o /tmp/tcs$v profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
$B -DPI2_TC_SPLITBAR=1 -DPI2_TC_TRACE -o /tmp/tcs1t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 64 130 1000 48; do
  for v in 0 1; do echo "== SPLITBAR=$v L=$L"; timeout 60 /tmp/tcs$v 3276800 $L | grep -E "tensor-core|hash|max|W "; done
done
for L in 100; do echo "== trace SPLITBAR=1 L=$L"; timeout 60 /tmp/tcs1t 3276800 $L | grep -E "SMSP"; done
echo "== small (C1-like rows)"; for v in 0 1; do timeout 60 /tmp/tcs$v 51200 100 | grep -E "tensor-core|hash"; done
