import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
kern = None; data = collections.OrderedDict()
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == 'Kernel Name':
        kern = r[1]; hdr = rows[i+1]; i += 2; data[kern] = (hdr, []); continue
    if kern and len(r) > 5: data[kern][1].append(r)
    i += 1
for k, (h, rs) in data.items():
    if len(sys.argv) > 2 and sys.argv[2] not in k: continue
    ie = h.index('Instructions Executed'); src = h.index('Source'); st = h.index('Warp Stall Sampling (All Samples)')
    agg = collections.Counter(); stall = collections.Counter(); tot = 0; tots = 0
    for r in rs:
        op = r[src].strip().split()
        if not op: continue
        o = op[0] if not op[0].startswith('@') else op[1]
        o = o.split('.')[0]
        n = float(r[ie] or 0); s = float(r[st] or 0)
        agg[o] += n; stall[o] += s; tot += n; tots += s
    print('==', k[:70], 'total warp inst %.3g' % tot)
    for o, n in agg.most_common(28): print(f'   {o:10s} {n/tot*100:5.1f}%  stall {stall[o]/max(tots,1)*100:5.1f}%')
