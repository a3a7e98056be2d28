# A/B of libs x ring depth (TSW_AB_DEPTH) on the bench workload
LIBS=${1:-"cur"}; CASES=${2:-"f64:8"}; ROUNDS=${3:-2}; DEPTHS=${4:-"4"}
for r in $(seq 1 $ROUNDS); do for L in $LIBS; do for d in $DEPTHS; do for c in $CASES; do
  dt=${c%%:*}; K=${c#*:}
  out=$(TSW_AB_DEPTH=$d TSW_LIB=abl/$L.so timeout 300 python tools/abtest.py $dt $K 2 2>&1 | tail -1)
  echo "{\"round\": $r, \"lib\": \"$L\", \"depth\": $d, \"case\": \"$c\", \"res\": $out}"
done; done; done; done
