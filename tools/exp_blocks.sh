summ() { python -c "
import sys,json
tot=0
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['h'], d['kern_ms'], d['err'], d['exact_share'], d['visits'])
    elif l.startswith('total'): print(l)
"; }
for mode in 0 1; do for ne in 0 1; do echo "== qblock_mode $mode no_eager $ne"; if [ $ne = 1 ]; then export FG_NO_EAGER=1; else unset FG_NO_EAGER; fi; FG_QBLOCK_MODE=$mode python tools/sweep_report.py --config 2 2>&1 | summ; done; done
unset FG_NO_EAGER
rm -f /tmp/dbg.bin; FG_QBLOCK_MODE=0 FG_DEBUG_BLOCKS=/tmp/dbg.bin python tools/sweep_report.py --config 2 > /dev/null 2>&1; python tools/block_stats.py /tmp/dbg.bin $(python -c "
import sys; sys.path.insert(0,'.')
import paper_1206_6857_b200 as fg
from paper_1206_6857_b200.configs import config
from paper_1206_6857_b200.summation_engine import query_block_count
wl=config(2); t=fg.build_tree(fg.PointStore(wl.references, wl.weights),25); print(query_block_count(t))")
