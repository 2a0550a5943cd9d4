# usage: bash scripts/probe/e2e_ab.sh -- e2e (host entry points) of the in-tree lib vs scripts/probe/variants/*.so
cd $GRAFT_REPO_ROOT
LIB=paper_2202_05977_b200/libkmd.so
cp $LIB /tmp/base.so
run() { timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 40 "$@" 2>&1 | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))"; }
for rep in 1 2; do
  echo "base: $(run) bf16 $(run --bf16)"
  for v in scripts/probe/variants/libkmd_*.so; do
    cp $v $LIB; touch -d '+1 hour' $LIB
    echo "$(basename $v): $(run) bf16 $(run --bf16)"
  done
  cp /tmp/base.so $LIB; touch -d '+1 hour' $LIB
done
