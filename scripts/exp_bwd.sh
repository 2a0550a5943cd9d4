cd $GRAFT_REPO_ROOT
python bench.py --mode bwd --steps 16 --warmup 4 > /dev/null 2>&1
for D in 0 1; do
KMD_DEBUG=$D timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:fused|bwd" -c 9 --csv --log-file gpurun_out/launches_bwd_$D.csv python bench.py --mode bwd --steps 16 --warmup 4 > /dev/null 2>&1
done
echo done
