for rl in 16 24 32 48 64; do echo "== ref_leaf $rl"; bash tools/sweep_short.sh --config 2 --ref-leaf $rl | tail -1; done
