cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mr.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_r2k.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2k.log
timeout 300 python bench.py --mode mr > gpurun_out/bench_r2k_mr.log 2>&1
bash scripts/exp_variants.sh > gpurun_out/var_r2k.log 2>&1
