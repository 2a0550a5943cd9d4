cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mr.py -m gpu -q -x > gpurun_out/pytest_r2l.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2l.log
timeout 300 python bench.py --mode mr --steps 200 --warmup 20 > gpurun_out/bench_r2l_mr.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r2l_mr.csv python bench.py --mode mr --steps 4 --warmup 3 > gpurun_out/ncu_r2l_mr.log 2>&1
