cd $GRAFT_REPO_ROOT
for M in 1 4; do for f in 0 1; do
  echo "== M=$M PI2_FUSED=$f"
  PI2_FUSED=$f python profiles/k_sweep.py --L 100 --M $M --min-log2 14 --max-log2 20 2>&1 | tail -4
done; done
