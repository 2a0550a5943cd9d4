# usage: bash scripts/gpu_ncu_mode.sh MODE TAG -- one ncu --set full capture of one step of a
# multi-kernel bench mode (bwd | mr | temporal), after the same command exits 0 without ncu
MODE=$1; TAG=$2
cd $GRAFT_REPO_ROOT
case $MODE in
  bwd) K='regex:lse_kernel|fused_tma|bwd_'; N=4 ;;
  mr) K='regex:down4|fused_tma|combine'; N=4 ;;
  temporal) K='regex:temporal'; N=1 ;;
esac
CMD="python bench.py --mode $MODE --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s $((2 * N)) -c $N -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_$TAG.log
tail -2 gpurun_out/ncu_full_$TAG.log
