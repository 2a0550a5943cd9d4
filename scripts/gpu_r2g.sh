cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2g.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2g.log
bash scripts/exp_variants.sh > gpurun_out/var_r2g.log 2>&1
