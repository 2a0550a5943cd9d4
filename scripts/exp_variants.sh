# usage: bash scripts/exp_variants.sh [extra bench args] -- bench the in-tree lib, then every
# scripts/probe/variants/libkmd_*.so (parity tests on each), restoring the in-tree lib after
cd $GRAFT_REPO_ROOT
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/libkmd_base.so
run() {
  timeout 120 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 "$@" 2>&1 | python -c "
import sys,json
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print((d.get('kernel_ms',{}).get('avg') or d.get('ms_per_step'))*1000 if d else 'FAIL', 'us', d.get('parity'))"
}
echo "base: $(run "$@")"
timeout 200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x 2>&1 | tail -1
for v in scripts/probe/variants/libkmd_*.so; do
  [ -e "$v" ] || continue
  cp $v $LIB; touch -d '+1 hour' $LIB
  echo "$(basename $v): $(run "$@")"
  timeout 200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x 2>&1 | tail -1
done
echo "base again: $(cp /tmp/libkmd_base.so $LIB; touch -d '+1 hour' $LIB; run "$@")"
