# chunk MMAs issued by converged warp 0 with elect.sync (PI2_TC_ELECT=1) vs thread 0 in a
# divergent branch (0); bitwise equal (hashes), harness times
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -DPI2_TC_ELECT=0 -o /tmp/tce0 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_ELECT=1 -o /tmp/tce1 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 1000; do for r in 1 2; do for v in 0 1; do
  echo "== ELECT=$v L=$L round $r"; timeout 60 /tmp/tce$v 3276800 $L | grep -E "tensor-core|hash"
done; done; done
