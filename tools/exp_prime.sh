for p in 0 0.5 0.2 0.1; do echo "== PRIME $p"; FG_PRIME_EPS=$p bash tools/sweep_short.sh --config 2 | tail -11; done
for p in 0.5 0.05; do echo "== C5 PRIME $p"; FG_PRIME_EPS=$p timeout 300 bash tools/sweep_short.sh --config 5 --sub 200 | tail -17; done
