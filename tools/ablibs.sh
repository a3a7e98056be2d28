# A/B timing of alternative library builds (abl/*.so via TSW_LIB), interleaved over rounds.
# usage: bash tools/ablibs.sh "v0 v1 v2" "f64:4 f32:8" ROUNDS
mkdir -p gpurun_out
LIBS=${1:-"v0 v1"}; CASES=${2:-"f64:4 f32:8"}; ROUNDS=${3:-2}
for r in $(seq 1 $ROUNDS); do
  for L in $LIBS; do
    for c in $CASES; do
      dt=${c%%:*}; K=${c#*:}
      out=$(TSW_LIB=abl/$L.so timeout 300 python tools/abtest.py $dt $K 2 2>&1 | tail -1)
      echo "{\"round\": $r, \"lib\": \"$L\", \"case\": \"$c\", \"res\": $out}"
    done
  done
done
