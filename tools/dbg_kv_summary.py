import collections, sys
for f in sys.argv[1:]:
    blocks=[]; cur=None
    for l in open(f):
        if l.startswith('run'):
            cur=[l.strip()]; blocks.append(cur)
        elif l.startswith('[dbg]') and cur is not None: cur.append(l)
    for blk in blocks:
        rows=[l.split() for l in blk[1:]]
        comp_in=collections.defaultdict(list); comp_done={}
        for r in rows:
            b=int(r[2]); w=r[3]; t=float(r[5])
            if w=='comp-in': comp_in[b].append((r[4],t))
            elif w=='comp-done': comp_done[b]=t
        ks=sorted(comp_done)
        wait_tot=0; prev=None; waits=[]
        for k in ks:
            ins=[t for _,t in comp_in.get(k,[])]
            inmax=max(ins) if ins else 0
            if prev is not None:
                w=max(0, inmax-prev); wait_tot+=w; waits.append(w)
            prev=comp_done[k]
        if ks: print(f.split('/')[-1], blk[0], '| computes', len(ks), 'span', round(comp_done[ks[-1]]-comp_done[ks[0]],2), 'input-wait', round(wait_tot,3), 'nonzero', sum(1 for w in waits if w>0.001), 'max', round(max(waits) if waits else 0,3))
