# DRAM bytes per kernel of a C2 / C4 device-noise iteration, fused (PI2_FUSED=1) vs unfused, without ncu's
# inter-kernel cache flush (--cache-control none), 3 iterations each
cd $GRAFT_REPO_ROOT
for fz in 1 0; do for c in C2 C4; do
  PI2_FUSED=$fz ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/fused${fz}_nocc_$c.csv python profiles/profile_step.py --config $c --iters 3 > /dev/null 2>&1
done; done
for fz in 1 0; do for c in C2 C4; do echo "## PI2_FUSED=$fz $c (per iteration, no cache flush)"; python profiles/dram_per_kernel.py gpurun_out/fused${fz}_nocc_$c.csv; done; done
