cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_bands.py tests/test_gpu_albedo.py tests/test_gpu_mr.py tests/test_gpu_checked.py -m gpu -q -x > gpurun_out/pytest_r2i.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2i.log
bash scripts/exp_variants.sh > gpurun_out/var_r2i.log 2>&1
