for b in 0 256 1024 4096; do echo "== BFS_CAP $b"; FG_BFS_CAP=$b bash tools/sweep_short.sh --config 2 | tail -11; done
for b in 0 1024; do echo "== C5 BFS_CAP $b"; FG_BFS_CAP=$b timeout 300 bash tools/sweep_short.sh --config 5 --sub 200 | tail -17; done
