cd $GRAFT_REPO_ROOT
for D in 0 34 66; do
  KMD_DEBUG=$D python bench.py --steps 800 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('debug=$D', round(d['kernel_ms']['avg']*1000,1), 'us')"
done
