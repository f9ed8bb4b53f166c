#!/bin/bash
# Alternate SINGLE-run timings (one bandwidth index per run) of engine variants
# on one box: tools/ab_runs.sh 5 "6 8 10" 6 cur v8   (config, bandwidth indices, plimit, variants)
cfg=$1; bws=$2; pl=$3; shift 3
for rep in 1 2; do
  for bw in $bws; do
    for v in "$@"; do
      if [ "$v" = cur ]; then lib=""; else lib="variants/$v.so"; fi
      ms=$(FG_LIB=$lib python tools/one_run.py --config $cfg --bw $bw --reps 3 --plimit $pl 2>/dev/null | awk '{print $3}')
      echo "C$cfg bw$bw plimit$pl $v $ms"
    done
  done
done
