# rollout_kernel (M = 1): rows of the next 1 or 2 steps in flight (PI2_ROLL1_AHEAD), A/B on one box.
# Build first:  for z in 1 2; do nvcc $F -DPI2_ROLL1_AHEAD=$z -I include -o _exp/ra$z.so paper_1503_00330_b200/csrc/pi2rh.cu; done
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in ra1 ra2; do
  cp _exp/$v.so paper_1503_00330_b200/_lib/libpi2rh.so
  for c in C4 C3; do
  python bench.py --config $c --steps 20 --no-cpu-baseline --no-north-star --no-other-configs 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v $c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done; done
