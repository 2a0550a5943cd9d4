cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/exp_variants.sh > gpurun_out/var_r2j.log 2>&1
