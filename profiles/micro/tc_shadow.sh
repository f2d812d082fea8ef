# LWPR shadow split (PI2_TC_SHADOW_SPLIT=1: finalize(t-1) in chunk 0's MMA shadow, features(t+1) in chunk 1's)
# vs both in chunk 0's (0): time and output bit hashes
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
for v in 0 1; do $B -DPI2_TC_SHADOW_SPLIT=$v -o /tmp/tcsh$v profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1; done
$B -DPI2_TC_SHADOW_SPLIT=1 -DPI2_TC_TRACE -o /tmp/tcsh1t profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200 130 64 1000; do for r in 1 2; do for v in 0 1; do echo "== SPLIT=$v L=$L round $r"; timeout 60 /tmp/tcsh$v 3276800 $L | grep -E "tensor-core|hash"; done; done; done
echo "== trace SPLIT=1 L=100"; timeout 60 /tmp/tcsh1t 3276800 100 | grep SMSP
