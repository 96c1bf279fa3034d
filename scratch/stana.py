import sys, json, numpy as np
d = json.load(open(sys.argv[1])); tr = np.array(d["trace"], dtype=np.int64)
t0 = tr[tr>0].min()
kb = np.load(sys.argv[2]); cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lo, hi = int(sys.argv[4]), int(sys.argv[5])
e = kb[cta]
for i in range(lo, hi):
    a, b, c = e[i]
    if a == 0: break
    print(i, "mma wait %.2f -> got +%.2f | issued %.2f (lat %.2f)" % ((a-t0)/1e3, (b-a)/1e3, (c-t0)/1e3, (b-c)/1e3))
