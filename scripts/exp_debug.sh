# role timing: KMD_DEBUG bits (kmd_tma.cu): 2 no exact path, 32 no field compute,
# 64 no fusion compute, 1024 no finalize, 1 no store
cd $GRAFT_REPO_ROOT
for D in ${DBG:-0 34 66 98 1090}; do
  KMD_DEBUG=$D python bench.py --steps 800 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('debug=$D', round(d['kernel_ms']['avg']*1000,1), 'us')"
done
