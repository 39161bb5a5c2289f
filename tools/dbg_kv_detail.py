import collections, sys
f=sys.argv[1]
blocks=[]; cur=None
for l in open(f):
    if l.startswith('run'): cur=[l.strip()]; blocks.append(cur)
    elif l.startswith('[dbg]') and cur is not None: cur.append(l)
blk=blocks[-1]
rows=[(l.split()[3], l.split()[4], float(l.split()[5]), int(l.split()[2])) for l in blk[1:]]
comp_done={b:t for w,s,t,b in rows if w=='comp-done'}
comp_in=collections.defaultdict(list)
for w,s,t,b in rows:
    if w=='comp-in': comp_in[b].append(t)
ks=sorted(comp_done); prev=None; shown=0
for k in ks:
    inmax=max(comp_in.get(k,[0]))
    if prev is not None and inmax-prev>0.05 and shown<6:
        shown+=1
        print(f"compute {k}: prev done {prev:.3f} inputs done {inmax:.3f} wait {inmax-prev:.3f}")
        ev=sorted([(t,w,s) for w,s,t,b in rows if prev-0.3<=t<=inmax+0.01 and w not in('comp-done','comp-in')])
        for t,w,s in ev: print(f"    {t:9.3f} {w:10s} {s}")
    prev=comp_done[k]
