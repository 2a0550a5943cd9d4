cd $GRAFT_REPO_ROOT
python bench.py --steps 400 --warmup 8 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('normal', round(d['kernel_ms']['avg']*1000,1), 'us')"
cp scripts/probe/libkmd_fastexp.so paper_2202_05977_b200/libkmd.so; touch -d '+1 hour' paper_2202_05977_b200/libkmd.so
python bench.py --steps 400 --warmup 8 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fastexp', round(d['kernel_ms']['avg']*1000,1), 'us', d['parity'])"
python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
