#!/bin/bash
# Alternate sweep timings of variants on one box: tools/ab.sh "2 5" base cur
# ("cur" = the in-tree build).  Prints config, variant, sweep kernel ms.
cfgs=$1; shift
for rep in 1 2; do
  for c in $cfgs; do
    for v in "$@"; do
      if [ "$v" = cur ]; then lib=""; else lib="variants/$v.so"; fi
      ms=$(FG_LIB=$lib python tools/one_sweep.py --config $c --reps $([ $c -le 2 ] && echo 8 || echo 3) 2>/dev/null | awk '{print $4}')
      echo "C$c $v $ms"
    done
  done
done
