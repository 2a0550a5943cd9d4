# usage: bash scripts/prof_debug.sh DEBUGBITS TAG
cd $GRAFT_REPO_ROOT
export KMD_DEBUG=$1
CMD="python bench.py --steps 16 --warmup 8 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_$2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 8 -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_$2.log 2>&1
echo "exit $?" >> gpurun_out/ncu_$2.log
