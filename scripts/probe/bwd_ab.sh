# usage: bash scripts/probe/bwd_ab.sh -- backward step time + backward tests: in-tree lib vs scripts/probe/variants/*.so
cd $GRAFT_REPO_ROOT
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/base.so
run() { timeout 300 python bench.py --mode bwd --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2))"; }
for rep in 1 2; do
  echo "base: $(run)"
  for v in scripts/probe/variants/libkmd_*.so; do
    cp $v $LIB; touch -d '+1 hour' $LIB
    echo "$(basename $v): $(run) $(timeout 300 python -m pytest tests/test_gpu_backward.py -q -x 2>&1 | tail -1)"
  done
  cp /tmp/base.so $LIB; touch -d '+1 hour' $LIB
done
