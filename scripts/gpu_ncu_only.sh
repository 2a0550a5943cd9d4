# usage: bash scripts/gpu_ncu_only.sh TAG -- the ncu part of scripts/gpu_final_r2.sh (launch list, full capture of the hot kernel, the bwd / mr / temporal steps)
TAG=$1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 16 --warmup 8 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused -c 40 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:fused -s 8 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu exit $?"
for mode in bwd mr temporal; do bash scripts/gpu_ncu_mode.sh $mode ${TAG}_$mode; done
