cd $GRAFT_REPO_ROOT
for v in scripts/probe/variants/libkmd_*.so; do echo "== $v"; timeout 120 python scripts/probe/dbg_variant.py $v; done > gpurun_out/dbg.log 2>&1
