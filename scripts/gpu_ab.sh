# usage: bash scripts/gpu_ab.sh TAG -- A/B of the in-tree lib against scripts/probe/variants/*.so
# (bench time + parity tests on each), logs in gpurun_out/var_TAG.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/exp_variants.sh > gpurun_out/var_$1.log 2>&1
