# usage: bash scripts/gpu_final_r2.sh TAG -- round-2 evidence: GPU tests, smoke, the default bench
# line, every other bench mode, the launch list + one ncu --set full capture of the hot kernel,
# ncu captures of the backward / MR / temporal steps and of the large-k (v1) kernel
TAG=${1:-r2}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
for m in "--height 720 --width 1280" "--albedo" "--bf16" "--mode mr" "--mode band" "--mode bwd" "--mode temporal" "--mode sweep" "--mode batch" "--impl reference --steps 3 --warmup 3"; do
  n=$(echo $m | tr -d ' -' )
  timeout 600 python bench.py $m 2>&1 | grep '^{' | tail -1 > gpurun_out/bench_${TAG}_$n.json
done
CMD="python bench.py --steps 16 --warmup 8 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused -c 40 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:fused -s 8 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_$TAG.log
for mode in bwd mr temporal; do bash scripts/gpu_ncu_mode.sh $mode ${TAG}_$mode; done
for k in 21 31; do
  timeout 300 python scripts/largek_case.py $k > gpurun_out/plain_${TAG}_k$k.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:fused_direct -s 2 -c 1 -o gpurun_out/prof_${TAG}_k$k python scripts/largek_case.py $k > gpurun_out/ncu_full_${TAG}_k$k.log 2>&1
  echo "exit $?" >> gpurun_out/ncu_full_${TAG}_k$k.log
done
