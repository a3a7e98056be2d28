# registers / spills / barriers of the temporally blocked kernels in a ptxas log
# usage: bash tools/ptxregs.sh [log] [pattern]
L=${1:-paper_2005_11931_b200/build_ptxas.log}; P=${2:-'k_step2d_tbI[df]Li(4|8|10)ELb0'}
grep -nE "Compiling entry function '_ZN3tsw11${P}" "$L" | while IFS=: read n rest; do
  name=$(echo "$rest" | grep -oE "k_step2d_tbI[^']*" | sed 's/EEEvNS_6TbArgsIT_EEi//')
  info=$(sed -n "$((n+1)),$((n+4))p" "$L" | grep -oE "[0-9]+ bytes spill stores|Used [0-9]+ registers|used [0-9]+ barriers" | tr '\n' ' ')
  echo "$name  $info"
done
