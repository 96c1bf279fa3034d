import json, sys, numpy as np
d = json.load(open(sys.argv[1]))
tasks = np.array(d["tasks"]); tr = np.array(d["trace"], dtype=np.int64)
types = tasks[:,0] & 0xff; ops = tasks[:,0] >> 8
t0 = tr[tr>0].min()
g = types == 0
print("stamps: 0 Bdep 1 tfull 5 pushed 2 cbarA 6 statsdone 3 cbarB 7 merged 4 done")
for o in range(ops[g].max()+1):
    sel = g & (ops == o)
    r = (tr[sel] - t0) / 1e3
    md = lambda a, b: np.median(r[:, b] - r[:, a])
    print(f"op {o:2d} n={sel.sum():3d} Bdep {r[:,0].min():7.1f} | tfull {md(0,1):5.1f} push {md(1,5):4.1f} barA {md(5,2):4.1f} stats {md(2,6):4.1f} barB {md(6,3):4.1f} merge {md(3,7):4.1f} apply+st {md(7,4):4.1f} | last {r[:,4].max():7.1f}")

if "trace2" in d:
    t2 = np.array(d["trace2"], dtype=np.int64)
    print("detail: apply | esync | stores | fence+esync | red")
    for o in range(ops[g].max()+1):
        sel = g & (ops == o)
        r = tr[sel]; q = t2[sel]
        print(f"op {o:2d} {np.median(q[:,4]-r[:,7])/1e3:4.2f} {np.median(q[:,5]-q[:,4])/1e3:4.2f} {np.median(q[:,6]-q[:,5])/1e3:4.2f} {np.median(q[:,7]-q[:,6])/1e3:4.2f} {np.median(r[:,4]-q[:,7])/1e3:4.2f}")

    cyc = (t2[g][:,1] - t2[g][:,0]).astype(float); ns = (t2[g][:,4] - tr[g][:,7]).astype(float)
    print("apply: median cycles", np.median(cyc), "median ns", np.median(ns), "=> MHz", np.median(cyc / ns * 1e3))
