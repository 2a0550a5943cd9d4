cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
timeout 600 python bench.py --mode mr --steps 200 --warmup 5 > gpurun_out/bench_mr.log 2>&1; echo "exit $?" >> gpurun_out/bench_mr.log
