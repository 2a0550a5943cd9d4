cd $GRAFT_REPO_ROOT
for S in 3,5,7,9,11,13 13,13,13,13,13,13 3,3,3,3,3,3 7,7,7,7,7,7 13,3,13,3,13,3 5; do
  python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 0 --sizes $S 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$S', round(d['kernel_ms']['avg']*1000,1), 'us', round(d['roofline']['frac'],3))"
done
