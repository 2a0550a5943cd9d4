cd $GRAFT_REPO_ROOT
for V in normal spin; do
  if [ $V = spin ]; then cp scripts/probe/libkmd_spin.so paper_2202_05977_b200/libkmd.so; touch -d '+1 hour' paper_2202_05977_b200/libkmd.so; fi
  for D in 0 1522; do
    KMD_DEBUG=$D python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$V debug=$D', round(d['kernel_ms']['avg']*1000,1), 'us')"
  done
done
