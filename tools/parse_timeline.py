import sys,re
calls=[];cur=None
for ln in sys.stdin:
    m=re.match(r"slot (\d+) chunk +(\d+)  h2d +([\d.]+)- +([\d.]+)  kernel - +([\d.]+)  d2h - +([\d.]+)",ln)
    if not m: continue
    ci=int(m.group(2)); v=[float(m.group(i)) for i in (3,4,5,6)]
    if ci==0: cur=[]; calls.append(cur)
    cur.append(v)
prev=None
for i,c in enumerate(calls):
    h2d=[b-a for a,b,_,_ in c]
    slow=[j for j,x in enumerate(h2d) if x>0.40]
    print(f"call {i}: start {c[0][0]:8.3f} period {'' if prev is None else round(c[0][0]-prev,3)} h2d mean {sum(h2d)/len(h2d):.3f} max {max(h2d):.3f} slow chunks {slow}")
    prev=c[0][0]
