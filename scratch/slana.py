import sys, json, numpy as np
d = json.load(open(sys.argv[1])); tr = np.array(d["trace"], dtype=np.int64)
t0 = tr[tr>0].min()
kb = np.load(sys.argv[2]); cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
e = kb[cta]
for i,(a,b,c) in enumerate(e):
    if a == 0 and c == 0: break
    print(i, "prod start %.2f  mma got B +%.2f  last A +%.2f" % ((a-t0)/1e3, (b-a)/1e3, (c-a)/1e3))
