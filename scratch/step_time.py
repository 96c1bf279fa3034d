"""Time one megakernel denoise step (S samples) alone; optional per-task trace dump."""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import _lib
from paper_2509_09560_b200 import diffusion as D
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfgname = sys.argv[2] if len(sys.argv) > 2 else "pusht"
trace_on = len(sys.argv) > 3 and sys.argv[3] == "trace"
cfg = D.PRESETS[cfgname]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=4)
P, G = torch.cuda.Stream(), torch.cuda.Stream()
sess = pol.open_session(capacity=2, lanes=S + 2, agents=1, max_outputs=4, max_frames=4, p_stream=P, g_stream=G)
lib = _lib.load()
for lane in range(S):
    sess.ingest(lane, lane, [pol.synthetic_observation(0, lane)])
sess.perceive(0, 0, 5)
slot, ver = sess.store.reserve(0)
sess.publish(0, 0, slot, ver)
torch.cuda.synchronize()
sess.fetch(0, 0)
ia = _lib.int_array
n = 0
if trace_on:
    n = lib.auras_unet_mega_trace(sess.plan, S, None, None, 0)
    tasks = np.zeros((n, 4), dtype=np.int32)
    trace = torch.zeros(n * 128 + 4096, dtype=torch.int64, device="cuda")
    assert lib.auras_unet_mega_trace(sess.plan, S, trace.data_ptr(), tasks.ctypes.data, n) == n
ts = []
for it in range(8):
    if trace_on:
        trace.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(G)
    _lib.check(lib.auras_unet_generate(sess.plan, S, ia(list(range(S))), ia([0] * S), ia([0] * S),
                                       ia([1] * S), 1, sess.R, sess.x.data_ptr(), _lib.ptr(sess.noise),
                                       sess.fetched.data_ptr(), 0, G.cuda_stream), "gen")
    e1.record(G)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("S", S, "step ms", " ".join(f"{t:.3f}" for t in ts), "min", min(ts[2:]))
x = sess.x[0, :S].cpu().numpy()
print("x finite", np.isfinite(x).all(), "x[0,:4]", x[0, :4])
if trace_on:
    tr = trace.cpu().numpy()
    np.savez(f"gpurun_out/ctrace_{S}.npz", tasks=tasks, trace=tr[:n * 128].reshape(n, 8, 16), cta=tr[n * 128:n * 128 + 296].reshape(148, 2))
