# usage: bash scripts/gpu_sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck /
# initcheck over scripts/sanitize_cases.py (every kernel family at small sizes); logs in gpurun_out/
TAG=${1:-r2}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1200 $CS --tool $tool $extra --kernel-name regex:kmd --print-limit 50 --error-exitcode 99 \
     python scripts/sanitize_cases.py > gpurun_out/sanitize_${TAG}_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_${TAG}_$tool.log
  tail -n 3 gpurun_out/sanitize_${TAG}_$tool.log
done
