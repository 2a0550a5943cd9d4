# usage: bash scripts/build_variant.sh NAME "EXTRA NVCC FLAGS"  -> scripts/probe/variants/libkmd_NAME.so
set -e
NAME=$1; shift
EXTRA="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/scripts/probe/variants
TMP=$(mktemp -d)
for f in $ROOT/paper_2202_05977_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 \
       --expt-relaxed-constexpr $EXTRA -I $ROOT/include -c $f -o $TMP/$(basename $f .cu).o || touch $TMP/FAILED &
done
wait
if [ -e $TMP/FAILED ]; then echo "build of $NAME failed"; rm -rf $TMP; exit 1; fi
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libkmd_$NAME.so $TMP/*.o -ldl
rm -rf $TMP
echo built $OUT/libkmd_$NAME.so
