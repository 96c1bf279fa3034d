"""Per-op phases of the sample-owned epilogue (cluster kernel trace, all ranks).
dep(0) act1(1) mmaend(2) drain-start(3, after tfull + rfree) pushed(4) landed(5) gn-done(8) stored(9) fenced(10) released(11)"""
import sys, numpy as np
d = np.load(sys.argv[1])
tasks, tr = d["tasks"], d["trace"].astype(np.int64)
types = tasks[:, 0] & 0xff; ops = tasks[:, 0] >> 8
g = types == 0
t0 = tr[g][:, :, 0][tr[g][:, :, 0] > 0].min()
r = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
pairs = [(0, 1, "act1"), (1, 2, "mma"), (2, 3, "tfull+rfree"), (3, 4, "push"), (4, 5, "land"), (5, 13, "sum"), (13, 6, "rfree"), (6, 7, "gn1"), (7, 8, "gn2"),
         (8, 9, "apply"), (9, 10, "fence"), (10, 11, "rel")]
print("op  n   dep0 " + " ".join(f"{n:>11s}" for _, _, n in pairs) + "   done")
for o in range(ops[g].max() + 1):
    sel = g & (ops == o)
    x = r[sel]
    ph = [np.nanmedian(x[:, :, b] - x[:, :, a]) for a, b, _ in pairs]
    print(f"{o:2d} {sel.sum():3d} {np.nanmin(x[:, :, 0]):6.1f} " + " ".join(f"{p:11.2f}" for p in ph) +
          f" {np.nanmax(x[:, :, 11]):6.1f}")
print("kernel span us:", np.nanmax(r[:, :, 11]) - np.nanmin(r[g][:, :, 0]))
