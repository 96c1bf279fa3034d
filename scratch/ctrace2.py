"""All-rank per-task trace of the cluster kernel (scratch/step_time.py S cfg trace)."""
import sys, numpy as np
d = np.load(sys.argv[1])
tasks, tr = d["tasks"], d["trace"].astype(np.int64)
types = tasks[:, 0] & 0xff; ops = tasks[:, 0] >> 8
g = types == 0
t0 = tr[g][tr[g] > 0].min()
r = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
names = ["dep", "act1", "mmaend", "tfull", "push", "barA", "stats", "barB", "merge", "apply", "fence", "rel"]
print("per op: first dep seen | median over (task,rank) of phase durations (us) | op done (max rel) | handoff to next op's first dep")
print("op    n  dep0   dep_spread " + " ".join(f"{n:>6s}" for n in ["act1", "mma", "tfull", "push", "barA", "stats", "barB", "merge", "apply", "fence", "rel"]) + "   done   hand")
prev_done = None
last = ops[g].max()
done_at = {}
for o in range(last + 1):
    sel = g & (ops == o)
    x = r[sel]                      # [tasks][8][16]
    dep = x[:, :, 0]
    done = np.nanmax(x[:, :, 11])
    done_at[o] = done
    ph = [np.nanmedian(x[:, :, k + 1] - x[:, :, k]) for k in range(11)]
    print(f"{o:2d} {sel.sum():4d} {np.nanmin(dep):6.1f} {np.nanmax(dep) - np.nanmin(dep):6.2f}   " +
          " ".join(f"{p:6.2f}" for p in ph) + f" {done:6.1f}")
# critical path: for each op, the time from the max done of its deps to its min dep-seen
cta = d["cta"]
print("kernel span us:", (np.nanmax(r[:, :, 11]) - np.nanmin(r[g][:, :, 0])))
