# full ncu captures (with source) of the non-LWPR kernels of a C2 iteration: rollout, attitude, partials
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}/r02"
mkdir -p "$OUT"
for k in rollout_group attitude partials; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o $OUT/${k}_c2 \
    python profiles/profile_step.py --iters 1 > $OUT/ncu_full_${k}.log 2>&1 || exit 1
done
echo done
