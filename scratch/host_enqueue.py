import os, sys, time, numpy as np, torch, cProfile, pstats
sys.path.insert(0, '.')
from paper_2509_09560_b200 import diffusion as D
from paper_2509_09560_b200 import _lib
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=4)
P, G = torch.cuda.Stream(), torch.cuda.Stream()
sess = pol.open_session(capacity=2, lanes=10, agents=1, max_outputs=4, max_frames=4, p_stream=P, g_stream=G)
torch.cuda.synchronize()
for it in range(3):
    t = time.perf_counter(); sess.perceive(0, 0, 5); h = time.perf_counter() - t
    torch.cuda.synchronize(); d = time.perf_counter() - t
    print(f"encoder: host enqueue {h*1e3:.2f} ms, to completion {d*1e3:.2f} ms")
lib = _lib.load()
item = [it for g in sess.encoder.groups.values() for it in g if it[0] == "conv"][3][1]
t = time.perf_counter()
for _ in range(100):
    lib.auras_conv(_lib.C.byref(item), sess.model.dt, 1, None, 0, sess.encoder.scratch.data_ptr(), sess.encoder.scratch.numel(), P.cuda_stream)
print("auras_conv host us", (time.perf_counter() - t) / 100 * 1e6)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): sess.perceive(0, 0, 5)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
