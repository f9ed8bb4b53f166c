#!/bin/bash
# Alternate sweep timings of the in-tree build under environment settings on
# one box: tools/ab_env.sh "2 5" "FG_FAR=0" "FG_FAR=1"
cfgs=$1; shift
for rep in 1 2; do
  for c in $cfgs; do
    for v in "$@"; do
      ms=$(env $v python tools/one_sweep.py --config $c --reps $([ $c -le 2 ] && echo 8 || echo 3) 2>/dev/null | awk '{print $4}')
      echo "C$c $v $ms"
    done
  done
done
