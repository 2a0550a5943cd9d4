cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 400 --warmup 8 --no-cpu-baseline --e2e-steps 0 --albedo > gpurun_out/bench_albedo.log 2>&1; echo "exit $?" >> gpurun_out/bench_albedo.log
