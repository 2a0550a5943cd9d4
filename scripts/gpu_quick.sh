cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 400 --warmup 8 > gpurun_out/bench_q.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_q.log
timeout 600 python bench.py --mode band --steps 50 --warmup 5 > gpurun_out/bench_band.log 2>&1; echo "band exit $?" >> gpurun_out/bench_band.log
