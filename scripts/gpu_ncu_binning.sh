# ncu --set full of the binning kernels of one 100-frame config-2 call (one GPU) -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/binprof_plain.log 2>&1 || exit 1
for k in block_masks radix_scatter tile_bounds prep_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/binprof_$k $CMD > gpurun_out/binprof_$k.log 2>&1; echo $k rc=$?
done
