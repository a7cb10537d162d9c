"""Phase costs from exit-at-phase variants (gpurun_out/gt_x1..x8, gt_default logs of scripts/gpu_ab2.sh)."""
import re
import sys

names = ['x1', 'x2', 'x3', 'x4', 'x5', 'x6', 'x7', 'x8', 'default']
d = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out'
data = {}
for n in names:
    for line in open(f'{d}/gt_{n}.log'):
        m = re.match(r'(\S+ \S+)\s+r=\s*(\d+).*compress\s+([\d.]+) us', line)
        if m:
            data.setdefault((m.group(1), int(m.group(2))), {})[n] = float(m.group(3))
labels = ['launch+wm', 'stream', 'B1', 'find', 'split', 'B2', 'fc', 'walk', 'cleanup']
print('case'.ljust(26) + ''.join(lb.rjust(10) for lb in labels) + '    total')
for key, v in data.items():
    prev, row = 0, []
    for n in names:
        row.append(v[n] - prev)
        prev = v[n]
    print(f'{key[0][:18]:18s} r={key[1]:<5d}' + ''.join(f'{x:10.2f}' for x in row) + f'{v["default"]:9.2f}')
