import csv, subprocess, sys
rep=sys.argv[1]; nenv=float(sys.argv[2]); top=int(sys.argv[3]) if len(sys.argv)>3 else 40
txt=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(txt.splitlines()))
cur=None; out=[]
for r in rows:
    if len(r)==2 and r[0]=="File Path": cur=r[1].split('/')[-1]; continue
    if len(r)>8 and r[0].isdigit():
        try: ti=int(r[8]); wi=int(r[7]); smp=int(r[4])
        except: continue
        out.append((wi,ti,smp,cur,int(r[0]),r[1][:110]))
tw=sum(o[0] for o in out); tt=sum(o[1] for o in out); ts=sum(o[2] for o in out)
print("warp inst/env %.0f thread inst/env %.0f samples %d"%(tw/nenv, tt/nenv, ts))
out.sort(reverse=True)
for o in out[:top]: print("%6.1f w/env %5.1f%%smp %s:%d | %s"%(o[0]/nenv,100*o[2]/ts,o[3],o[4],o[5]))
