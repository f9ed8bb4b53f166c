# compact sweep summary: h, kernel ms, err, exact share, visits
python tools/sweep_report.py "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['h'], d['kern_ms'], d['err'], d['exact_share'], d['fp32_share'], d['visits'], d['dh'], d.get('naive_ms',''))
    else: print(l)
"
