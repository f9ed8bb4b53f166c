# FG_DEBUG_SWEEP launch time vs summed task cycles for C2/C3: full sweep vs a 1/8 query-block shard
mkdir -p gpurun_out
for c in 2 3; do
FG_DEBUG_SWEEP=1 timeout 200 python - $c <<'PY' >> gpurun_out/floor.log 2>&1
import sys, torch, paper_1206_6857_b200 as fg
from paper_1206_6857_b200.configs import config
from paper_1206_6857_b200.summation_engine import query_block_count
wl = config(int(sys.argv[1])); t = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
hs = list(wl.bandwidths); cfg = fg.RunConfig(bandwidth=hs[0], epsilon=wl.epsilon)
nb = query_block_count(t); out = torch.zeros(len(hs), wl.m, dtype=torch.float64, device="cuda")
for br in [None, None, (0, nb, 8), (0, nb, 8)]:
    print(wl.name, "block_range", br, file=sys.stderr, flush=True)
    fg.sweep_run(cfg, t, t, hs, out=out, block_range=br)
PY
done
cat gpurun_out/floor.log
