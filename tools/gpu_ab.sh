# A/B of alternative builds: bitwise TB tests on each, then interleaved timing
# usage: bash tools/gpu_ab.sh "v0 v1 v2" "f64:8 f32:8" ROUNDS
mkdir -p gpurun_out
LIBS=${1:-"v0 v1"}; CASES=${2:-"f64:8 f32:8"}; ROUNDS=${3:-3}
for L in $LIBS; do
  TSW_LIB=abl/$L.so timeout 600 python -m pytest tests/test_tblock_gpu.py -q -x -p no:cacheprovider > gpurun_out/ab_test_$L.log 2>&1
  echo "tests $L rc=$? $(tail -1 gpurun_out/ab_test_$L.log)"
done
bash tools/ablibs.sh "$LIBS" "$CASES" $ROUNDS
