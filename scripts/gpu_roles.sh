# usage: bash scripts/gpu_roles.sh TAG -- role isolation (KMD_DEBUG bits, exp_debug.sh) for every
# scripts/probe/variants/*.so built with -DKMD_DEBUG_SWITCHES; logs in gpurun_out/roles_TAG.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/base.so
for v in scripts/probe/variants/libkmd_*.so; do
  cp $v $LIB; touch -d '+1 hour' $LIB
  echo "== $(basename $v)" >> gpurun_out/roles_$1.log
  DBG="${DBG:-0 66 482}" bash scripts/exp_debug.sh >> gpurun_out/roles_$1.log 2>&1
done
cp /tmp/base.so $LIB; touch -d '+1 hour' $LIB
