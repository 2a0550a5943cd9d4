cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 16 --warmup 8 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_r2f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:fused -s 8 -c 1 -o gpurun_out/prof_r2f $CMD > gpurun_out/ncu_full_r2f.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_r2f.log
bash scripts/exp_variants.sh > gpurun_out/var_r2f.log 2>&1
