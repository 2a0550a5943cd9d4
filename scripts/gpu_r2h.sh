cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_backward.py tests/test_gpu_bands.py -m gpu -q -x > gpurun_out/pytest_r2h.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2h.log
bash scripts/exp_variants.sh > gpurun_out/var_r2h.log 2>&1
