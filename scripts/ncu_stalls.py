import csv, subprocess, sys
rep=sys.argv[1]
txt=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(txt.splitlines()))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
cols=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot={c:0 for c in cols}
top=[]
for r in rows[2:]:
    try:
        for c in cols: tot[c]+=int(r[idx[c]] or 0)
        top.append((int(r[idx['Warp Stall Sampling (All Samples)']]), r[1][:60], {c:int(r[idx[c]] or 0) for c in cols}))
    except: pass
s=sum(tot.values())
for c,v in sorted(tot.items(), key=lambda x:-x[1])[:10]: print("%-28s %5.1f%%"%(c,100*v/s))
top.sort(key=lambda x:-x[0])
for t in top[:int(sys.argv[2]) if len(sys.argv)>2 else 15]:
    mx=max(t[2].items(), key=lambda x:x[1])
    print("%6d %-60s %s"%(t[0],t[1],mx))
