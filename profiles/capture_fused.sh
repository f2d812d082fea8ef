# ncu --set full of the fused step kernel (C2 and C4 device-noise iterations)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT="${OUT:-gpurun_out}/r02"
mkdir -p "$OUT"
for c in C2 C4; do
  ncu --set full --clock-control none --import-source on -k regex:fused_step -c 1 -f -o $OUT/fused_$c \
    python profiles/profile_step.py --config $c --iters 1 > $OUT/ncu_full_fused_$c.log 2>&1 || exit 1
done
echo done
