# bench the in-tree lib and every variant (no parity tests: for probes that change results)
cd $GRAFT_REPO_ROOT
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/libkmd_base.so
run() { timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 "$@" 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print(round(d['kernel_ms']['avg']*1000,2), 'us')"; }
echo "base: $(run "$@")"
for v in scripts/probe/variants/libkmd_*.so; do
  cp $v $LIB; touch -d '+1 hour' $LIB
  echo "$(basename $v): $(run "$@")"
done
cp /tmp/libkmd_base.so $LIB; touch -d '+1 hour' $LIB
