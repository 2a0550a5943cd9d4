cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2d.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2d.log
bash scripts/exp_variants.sh > gpurun_out/var_r2d.log 2>&1
