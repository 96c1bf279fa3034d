"""Per-task timeline of one megakernel denoise step (S samples), no other streams running."""
import sys, json, numpy as np, torch, ctypes as C
sys.path.insert(0, '.')
from paper_2509_09560_b200 import _lib
from paper_2509_09560_b200 import diffusion as D
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = D.PRESETS["pusht"]
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
n = lib.auras_unet_mega_trace(sess.plan, S, None, None, 0)
tasks = np.zeros((n, 4), dtype=np.int32)
trace = torch.zeros(n * 8 + 148 * 1024 * 3, dtype=torch.int64, device="cuda")
assert lib.auras_unet_mega_trace(sess.plan, S, trace.data_ptr(), tasks.ctypes.data, n) == n
batch = [(l, 0, 1) for l in range(S)]
sess.gen.__dict__  # noqa
import dataclasses
sess.gen = dataclasses.replace(sess.gen, use_graph=False) if False else sess.gen
for it in range(3):
    trace.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(G)
    ia = _lib.int_array
    _lib.check(lib.auras_unet_generate(sess.plan, S, ia([b[0] for b in batch]), ia([0] * S), ia([0] * S),
                                       ia([1] * S), 1, sess.R, sess.x.data_ptr(), _lib.ptr(sess.noise),
                                       sess.fetched.data_ptr(), 0, G.cuda_stream), "gen")
    e1.record(G)
    torch.cuda.synchronize()
    print("step ms", e0.elapsed_time(e1))
full = trace.cpu().numpy()
tr = full[:n * 8].reshape(n, 8)
kbt = full[n * 8:].reshape(148, 1024, 3)
t0 = tr[tr > 0].min()
types = tasks[:, 0] & 0xff
ops = tasks[:, 0] >> 8
out = {"S": S, "tasks": tasks.tolist(), "trace": (np.where(tr > 0, tr - t0, -1)).tolist()}
np.save("gpurun_out/kbtrace.npy", np.where(kbt > 0, kbt - t0, -1))
json.dump(out, open("gpurun_out/mega_trace.json", "w"))
print("ops", ops.max() + 1)
for o in range(ops.max() + 1):
    g = (types == 0) & (ops == o)
    e = (types == 1) & (ops == o)
    gb0 = tr[g, 0] - t0; gd1 = tr[g, 3] - t0; ee0 = tr[e, 0] - t0; ee1 = tr[e, 1] - t0
    f = lambda col: (tr[g, col] - t0) / 1e3
    print(f"op {o:2d}: n={g.sum():3d} Bdep {f(0).min():6.1f} Blast {np.median(f(1)-f(0)):5.1f} | mma0 {np.median(f(4)-f(0)):5.1f} A0 {np.median(f(5)-f(0)):5.1f} B0 {np.median(f(6)-f(0)):5.1f} commit {np.median(f(7)-f(0)):5.1f} (max {np.max(f(7)-f(0).min()):5.1f}) drain0 {np.median(f(2)-f(0)):5.1f} drained {np.median(f(3)-f(0)):5.1f} (max {np.max(f(3))-f(0).min():5.1f}) | epi {(ee0.min()-gd1.max())/1e3:4.1f} dur {(ee1.max()-ee0.min())/1e3:5.1f}")
print("EPI breakdown (us from gate): stats1 stats2 stores end")
for o in range(ops.max() + 1):
    e = (types == 1) & (ops == o)
    g0 = tr[e, 0]
    f = lambda c: np.median((tr[e, c] - g0) / 1e3)
    print(f"  op {o:2d}: {f(2):5.2f} {f(3):5.2f} {f(4):5.2f} {f(1):5.2f}")
