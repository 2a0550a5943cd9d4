# usage: bash scripts/gpu_quick.sh TAG -- GPU tests + a short default bench (no ncu)
TAG=${1:-q}
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log; python - <<'PY' gpurun_out/bench_$TAG.log
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print("BENCH", d["value"], "us", d["kernel_ms"]["avg"]*1e3, "frac", d["roofline"]["frac"])
PY
if [ -n "$ALL" ]; then
for m in "--albedo" "--bf16" "--mode mr" "--mode band" "--mode bwd" "--mode temporal"; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 0 $m 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('$m', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step']*1e3,1), 'us')"
done
fi
