"""Act/MMA-side detail of the cluster-kernel trace: dep seen -> first act TMA issued (13)
-> MMA warp enters task (15) -> weights ready (14) -> first act box landed (1)."""
import sys, numpy as np
d = np.load(sys.argv[1])
tasks, tr = d["tasks"], d["trace"].astype(np.int64)
types = tasks[:, 0] & 0xff; ops = tasks[:, 0] >> 8
g = types == 0
t0 = tr[g][tr[g] > 0].min()
r = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
print("op  dep->issued  dep->syncwarp  dep->emptyB_ok  dep->act1  (medians us)")
for o in range(ops[g].max() + 1):
    x = r[g & (ops == o)]
    f = lambda k: np.nanmedian(x[:, :, k] - x[:, :, 0])
    print(f"{o:2d} {f(13):8.2f} {f(15):10.2f} {f(14):10.2f} {f(1):8.2f}")
print("emptyB already complete at first wait (1) / not (2):", np.unique(tr[g][:, :, 13], return_counts=True))
