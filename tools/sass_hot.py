"""Summarise an `ncu --page source --csv` SASS dump: hottest instructions by stall samples."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = next(x for x in r if 'Source' in x and 'Address' in x)
si, ws, ie = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
rows = [x for x in r if len(x) > ie and x[0].startswith('0x')]
tot = sum(float(x[ws]) for x in rows)
toti = sum(float(x[ie]) for x in rows)
print(f'samples {tot:.0f} instructions {toti:.0f} sass_lines {len(rows)}')
for x in sorted(rows, key=lambda x: -float(x[ws]))[:top]:
    print(f"{float(x[ws]):7.0f} {float(x[ie]):9.0f}  {x[si].strip()[:100]}")
