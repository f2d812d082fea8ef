cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 1 0; do
  for c in C2 C4 C5; do
  PI2_STORE_Z=$v python bench.py --config $c --steps 20 --no-cpu-baseline --no-north-star --no-other-configs 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('z$v $c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done; done
