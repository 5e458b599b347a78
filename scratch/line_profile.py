"""Per-source-line executed instructions / stall samples: joins ncu's SASS
source page (csv) with nvdisasm -g line info of the same cubin.
usage: line_profile.py sass.csv dis.txt kernel_substr mangled_substr"""
import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
dis = open(sys.argv[2]).read().split('\n')
kname, mname = sys.argv[3], sys.argv[4]
# ncu side
data = None; i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == 'Kernel Name':
        if kname in r[1] and data is None:
            hdr = rows[i + 1]; data = []; i += 2
            while i < len(rows) and not (rows[i] and rows[i][0] == 'Kernel Name'):
                if len(rows[i]) > 5: data.append(rows[i])
                i += 1
            break
    i += 1
ai, ie, st = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
base = int(data[0][ai], 16)
# disasm side
in_fn = False; line = None; off2line = {}; file = None
for l in dis:
    if l.startswith('//---------------------'):
        in_fn = mname in l; continue
    if not in_fn: continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m: file, line = m.group(1).split('/')[-1], int(m.group(2)); continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m: off2line[int(m.group(1), 16)] = (file, line)
agg = collections.Counter(); sta = collections.Counter(); tot = 0; tots = 0
for r in data:
    off = int(r[ai], 16) - base
    key = off2line.get(off, ('?', 0))
    n = float(r[ie] or 0); s = float(r[st] or 0)
    agg[key] += n; sta[key] += s; tot += n; tots += s
print('total warp inst %.4g, stall samples %d' % (tot, tots))
for k, n in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 45]:
    print(f'{k[0]:22s}:{k[1]:4d}  inst {n/tot*100:5.1f}%  stall {sta[k]/tots*100:5.1f}%')
if len(sys.argv) > 6:
    regions = [tuple(x.split(':')) for x in sys.argv[6].split(',')]  # name:lo-hi
    ra = collections.Counter(); rs = collections.Counter()
    for k, n in agg.items():
        name = 'other'
        for nm, rng in regions:
            lo, hi = map(int, rng.split('-'))
            if lo <= k[1] <= hi and True: name = nm
        ra[name] += n; rs[name] += sta[k]
    for nm, n in ra.most_common(): print(f'{nm:12s} inst {n/tot*100:5.1f}%  stall {rs[nm]/tots*100:5.1f}%  thread-inst/pp {n*32/537e6:6.1f}')
