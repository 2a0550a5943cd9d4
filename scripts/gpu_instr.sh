# usage: bash scripts/gpu_instr.sh -- per-role wait breakdown (KMD_INSTR builds in scripts/probe/instr/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in scripts/probe/instr/*.so; do
  n=$(basename $v .so)
  nw=12; case $n in *vsplit*) nw=16 ;; esac
  NWARPS=$nw timeout 300 python scripts/probe/run_instr.py $v > gpurun_out/$n.log 2>&1
done
