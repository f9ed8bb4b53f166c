"""Register-liveness histogram of one kernel from `nvdisasm -plr -lrm count` output."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split('\n')
name = sys.argv[2]
start = next(i for i, l in enumerate(lines) if (name + ':') in l and not l.strip().startswith('.'))
end = start + 1
while end < len(lines) and not lines[end].strip().startswith('.section'):
    end += 1
counts = []
for l in lines[start:end]:
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);.*?\|\s*(\d+)', l)
    if m:
        counts.append((int(m.group(3)), m.group(1), m.group(2)[:60]))
print(sorted(counts, reverse=True)[:6])
hist = collections.Counter(c // 8 * 8 for c, _, _ in counts)
print(sorted(hist.items()))
