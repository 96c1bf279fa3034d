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
    n = 200
    buf = (ctypes.c_longlong * n)()
    m = _lib.load().auras_dpt_persist_trace(den.pplan, buf, n)
    t = np.array(buf[:m], dtype=np.int64)
    d = np.diff(t) / 1e3
    kinds = []
    print("phases", m - 1, "total us", (t[-1] - t[0]) / 1e3)
    print("per phase us:", " ".join(f"{x:.1f}" for x in d))
