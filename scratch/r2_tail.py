"""Inter-iteration tail of the cluster kernel: per-iteration marginal time
(count 13 vs 1 in one launch) against the single-iteration op-chain span
from the per-task trace (op 0 dependency seen -> last op released)."""
import sys, numpy as np, torch
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
ia = _lib.int_array


def run(count, trace=None):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(G)
    _lib.check(lib.auras_unet_generate(sess.plan, S, ia(list(range(S))), ia([0] * S), ia([0] * S),
                                       ia([count] * S), 1, sess.R, sess.x.data_ptr(), _lib.ptr(sess.noise),
                                       sess.fetched.data_ptr(), 0, G.cuda_stream), "gen")
    e1.record(G)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


res = {}
for c in (1, 2, 13):
    ts = [run(c) for _ in range(8)]
    res[c] = min(ts[2:])
    print(f"count {c:2d}: launch ms min {res[c]:.4f}  all {' '.join(f'{t:.3f}' for t in ts)}")
print(f"marginal per iteration (13 vs 1): {(res[13] - res[1]) / 12 * 1e3:.1f} us; (2 vs 1): {(res[2] - res[1]) * 1e3:.1f} us")
n = lib.auras_unet_mega_trace(sess.plan, S, None, None, 0)
tasks = np.zeros((n, 4), dtype=np.int32)
trace = torch.zeros(n * 128 + 4096, dtype=torch.int64, device="cuda")
assert lib.auras_unet_mega_trace(sess.plan, S, trace.data_ptr(), tasks.ctypes.data, n) == n
for _ in range(3):
    trace.zero_()
    run(1)
tr = trace.cpu().numpy()[:n * 128].reshape(n, 8, 16).astype(np.int64)
types = tasks[:, 0] & 0xff
ops = tasks[:, 0] >> 8
g = types == 0
t0 = tr[g][:, :, 0][tr[g][:, :, 0] > 0].min()
last = ops[g].max()
done_last = tr[g & (ops == last)][:, :, 11].max()
fin = tr[types == 3]
print(f"single iteration: op 0 dep -> last op released {(done_last - t0) / 1e3:.1f} us")
fv = fin[:, :, 11][fin[:, :, 11] > 0]
fs = fin[:, :, 0][fin[:, :, 0] > 0]
print(f"final tasks: first spin-done {(fs.min() - t0) / 1e3:.1f} us, last end {(fv.max() - t0) / 1e3:.1f} us (S = {S})")
