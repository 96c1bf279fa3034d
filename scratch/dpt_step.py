"""Time one DP-T denoise iteration over S samples through the session (graph replay),
and the sum of its kernel durations under ncu when run with `ncu` (argv[2] = 'once')."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import diffusion as D
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
once = len(sys.argv) > 2 and sys.argv[2] == "once"
cfg = D.PRESETS["vit_dpt"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=4)
P, G = torch.cuda.Stream(), torch.cuda.Stream()
sess = pol.open_session(capacity=2, lanes=S + 2, agents=1, max_outputs=4, max_frames=4, p_stream=P, g_stream=G)
for lane in range(S):
    sess.ingest(lane, lane, [pol.synthetic_observation(0, lane)])
sess.perceive(0, 0, len(pol.perception.layers))
slot, ver = sess.store.reserve(0)
sess.publish(0, 0, slot, ver)
torch.cuda.synchronize()
sess.fetch(0, 0)
batch = [(lane, 10 * lane, 1) for lane in range(S)]
for _ in range(3):
    sess.generate(batch)
torch.cuda.synchronize()
if once:
    sess.generate(batch)
    torch.cuda.synchronize()
    sys.exit(0)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(G)
    sess.generate(batch)
    e1.record(G)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("S", S, "dpt iteration ms", " ".join(f"{t:.3f}" for t in ts), "min", min(ts))
if os.environ.get("AURAS_DPT_TRACE"):
    import ctypes
    from paper_2509_09560_b200 import _lib
    den = sess.denoiser
    n = 20000
    buf = (ctypes.c_longlong * n)()
    mm = _lib.load().auras_dpt_persist_trace(den.pplan, buf, n)
    n_ops = (mm - 1) // 73
    m = n_ops + 1
    t = np.array(buf[:m], dtype=np.int64)
    sub = np.array(buf[m:9 * n_ops + 1], dtype=np.int64).reshape(n_ops, 8)
    ks = np.array(buf[9 * n_ops + 1:mm], dtype=np.int64).reshape(n_ops, 64)
    d = np.diff(t) / 1e3
    kinds = []
    print("phases", m - 1, "total us", (t[-1] - t[0]) / 1e3)
    print("per phase us:", " ".join(f"{x:.1f}" for x in d))
    names = ["start", "prod", "ln", "mma0", "mmaN", "done", "epi", "fence"]
    print("sub-phase clocks (cycles after phase start; layer 2 ops + head/update):")
    for oi in list(range(7, 13)) + [n_ops - 1]:
        r = sub[oi]
        print(f"  op {oi:3d}: " + " ".join(f"{names[k]}={(r[k] - r[0]) if r[k] else -1}" for k in range(1, 8)))
    for oi in (7, 9, 11, 12, n_ops - 1):
        r0 = sub[oi][0]
        print(f"  op {oi} epilogue : " + " ".join(str(ks[oi][48 + j] - r0) if ks[oi][48 + j] else "-" for j in range(6)))
        k = ks[oi]
        for name, off in (("B ready", 0), ("A issued", 16), ("MMA full", 32)):
            print(f"  op {oi} {name:9s}: " + " ".join(str(k[off + j] - r0) if k[off + j] else "-" for j in range(16)))
    for oi in (9, 10, 12, 13, 15):
        r0 = sub[oi][0]
        print(f"  op {oi} attn-scores/attn-end/ln-landed: {ks[oi][56] - r0 if ks[oi][56] else '-'} {ks[oi][57] - r0 if ks[oi][57] else '-'}")
    for oi in range(n_ops):
        if ks[oi][60] and sub[oi][0]:
            r0 = sub[oi][0]
            print(f"  op {oi} xattn enter/staged/synced/scored/stored: " +
                  " ".join(str(ks[oi][56 + j] - r0) if ks[oi][56 + j] else "-" for j in (4, 0, 1, 2, 3)))
            break
