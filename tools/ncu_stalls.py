import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]
ix={h:i for i,h in enumerate(hdr)}
data=rows[2:]
S="Warp Stall Sampling (All Samples)"
tot=sum(float(r[ix[S]] or 0) for r in data)
print("total samples", tot)
reasons=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg={h:sum(float(r[ix[h]] or 0) for r in data) for h in reasons}
print(' '.join(f'{h[6:]}:{v:.0f}' for h,v in sorted(agg.items(), key=lambda x:-x[1]) if v>0))
n=int(sys.argv[2]) if len(sys.argv)>2 else 45
top=sorted(data,key=lambda r:-float(r[ix[S]] or 0))[:n]
for r in top:
    rs=sorted(((float(r[ix[h]] or 0),h[6:]) for h in reasons), reverse=True)[:3]
    print(r[ix["Address"]][-5:], f'{float(r[ix[S]]):6.0f}', f'{r[ix["Instructions Executed"]]:>6}', r[ix["Source"]][:60].ljust(60), ' '.join(f'{n}:{v:.0f}' for v,n in rs if v>0))
