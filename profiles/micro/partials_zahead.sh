# partials_kernel: stored-normal loads PI2_PARTIALS_ZAHEAD elements ahead (0 / 2 / 4), A/B on one box.
# Build the three libraries first (here, nvcc cross-compiles):
#   F=$(python -c "from paper_1503_00330_b200 import _build as b; print(' '.join(b.NVCC_FLAGS))")
#   for z in 0 2 4; do nvcc $F -DPI2_PARTIALS_ZAHEAD=$z -I include -o _exp/pz$z.so paper_1503_00330_b200/csrc/pi2rh.cu; done
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in pz0 pz2 pz4; do
  cp _exp/$v.so paper_1503_00330_b200/_lib/libpi2rh.so
  for c in C2 C4; do
  python bench.py --config $c --steps 30 --no-cpu-baseline --no-north-star --no-other-configs 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v $c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done; done
