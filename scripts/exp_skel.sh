cd $GRAFT_REPO_ROOT
for S in 3 3,3 3,3,3 3,3,3,3,3,3; do
  for D in 1522 0; do
    KMD_DEBUG=$D python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 --sizes $S 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sizes=$S debug=$D', round(d['kernel_ms']['avg']*1000,1), 'us')"
  done
done
python - <<'PY'
import torch
x = torch.empty(1, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(10): x.add_(1)
ts=[]
for _ in range(100):
    s.record(); x.add_(1); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e)*1000)
print("tiny torch kernel event time us: median", sorted(ts)[50])
PY
