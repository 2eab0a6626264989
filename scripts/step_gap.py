import csv,sys
rows = sorted((int(r[0]), int(r[1]), int(r[4]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1])) if len(r) >= 6)
g=[i for i,r in enumerate(rows) if 'gather_kernel' in r[3]]
out=[]
for kb in range(1,8):
    lo=g[-1-kb]; t0=rows[lo][0]
    nxt=min(r[0] for r in rows[lo+1:lo+10])
    prev=max(r[1] for r in rows[lo-6:lo])
    out.append(f"gather {(rows[lo][1]-t0)/1e3:.1f}us, next start {(nxt-t0)/1e3:.1f}, prev end {(prev-t0)/1e3:.1f}")
print("\n".join(out))
