# partials_kernel: ZAHEAD x MINB A/B (second pass).  Build first:
#   for v in "2 0" "3 4" "4 4" "3 0"; do set -- $v; nvcc $F -DPI2_PARTIALS_ZAHEAD=$1 -DPI2_PARTIALS_MINB=$2 -I include -o _exp/pa$1$2.so paper_1503_00330_b200/csrc/pi2rh.cu; done
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in pa20 pa34 pa44 pa30; do
  cp _exp/$v.so paper_1503_00330_b200/_lib/libpi2rh.so
  for c in C2 C4; do
  python bench.py --config $c --steps 30 --no-cpu-baseline --no-north-star --no-other-configs 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v $c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done; done
