cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|down|combine" -c 20 --csv --log-file gpurun_out/launches_r2m_mr.csv python bench.py --mode mr --steps 4 --warmup 3 > gpurun_out/ncu_r2m_mr.log 2>&1
