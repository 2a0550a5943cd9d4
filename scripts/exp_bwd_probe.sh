# backward pass-A probes: bwd bench with the in-tree lib and each variant, KMD_DEBUG in {0, 1}
cd $GRAFT_REPO_ROOT
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/libkmd_base.so
run() { timeout 300 python bench.py --mode bwd --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print(round(d['ms_per_step']*1000,1), 'us')"; }
for d in 0; do echo "base debug=$d: $(KMD_DEBUG=$d run)"; done
for v in scripts/probe/variants/libkmd_*.so; do
  cp $v $LIB; touch -d '+1 hour' $LIB
  for d in 0; do echo "$(basename $v) debug=$d: $(KMD_DEBUG=$d run)"; done
done
cp /tmp/libkmd_base.so $LIB; touch -d '+1 hour' $LIB
