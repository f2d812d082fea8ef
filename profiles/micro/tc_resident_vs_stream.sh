# resident weights (default where they fit) vs TMA-streamed (PI2_LWPR_TC_STREAM=1) with the unrolled loop
cd $GRAFT_REPO_ROOT
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1503_00330_b200/csrc"
$B -o /tmp/tct profiles/micro/lwpr_tc_test.cu || exit 1
for r in 1 2; do
  for L in 100 200; do
    echo "L=$L resident: $(timeout 60 /tmp/tct 3276800 $L | grep -E 'tensor-core' | tr '\n' ' ')"
    echo "L=$L streamed: $(PI2_LWPR_TC_STREAM=1 timeout 60 /tmp/tct 3276800 $L | grep -E 'tensor-core' | tr '\n' ' ')"
  done
done
