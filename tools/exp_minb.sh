for mb in 4 5 6 8; do echo "== MINB $mb"; FG_TRAV_MINB=$mb bash tools/sweep_short.sh --config 2 | tail -6; done
