# experiment: two 32-field TMEM item buffers with a named-barrier handoff (PI2_TC_DB=1, PI2_TC_CHUNK=32) vs the
# product (64-field chunks, one buffer) and the one-buffer body at 32-field chunks
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -o /tmp/tdb_base profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_CHUNK=32 -o /tmp/tdb_c32 profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_CHUNK=32 -DPI2_TC_DB=1 -o /tmp/tdb_db profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
$B -DPI2_TC_CHUNK=32 -DPI2_TC_DB=1 -DPI2_TC_TRACE -o /tmp/tdb_dbt profiles/micro/lwpr_tc_test.cu 2>/dev/null || exit 1
for L in 100 200; do for v in base c32 db; do echo "== $v L=$L"; timeout 60 /tmp/tdb_$v 3276800 $L | grep -E "tensor-core|max"; done; done
echo "== trace db L=100"; timeout 60 /tmp/tdb_dbt 3276800 100 | grep -E "SMSP|  w0[0-9]" | head -60
