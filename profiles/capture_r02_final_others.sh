#!/bin/bash
# Full ncu captures of the non-LWPR kernels at C2 or C4 (end of round 2): bash this C2|C4
# (one config per gpurun call: the reports of both exceed gpurun's 64 MiB copy-back).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}/r02f"
mkdir -p "$OUT"
cfg=${1:-C2}
if [ "$cfg" = C2 ]; then ks="rollout_group attitude partials combine"; else ks="rollout_kernel attitude combine"; fi
for k in $ks; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o $OUT/${k}_${cfg,,} \
    python profiles/profile_step.py --config $cfg --iters 1 > $OUT/ncu_full_${k}_${cfg,,}.log 2>&1 || exit 1
done
echo done
