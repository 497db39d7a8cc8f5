# median of each host phase over 12 runs
GN_HOST_TIMING=1 python tools/host_ab.py 2>&1 >/dev/null | python -c "
import sys, collections, statistics
d = collections.defaultdict(list)
for line in sys.stdin:
    if line.startswith('[gn host]'):
        parts = line[9:].rsplit(None, 2)
        d[parts[0].strip()].append(float(parts[1]))
for k, v in d.items():
    if len(v) > 2: print(f'{k:32s} median {statistics.median(v[2:]):7.2f} ms')
"
