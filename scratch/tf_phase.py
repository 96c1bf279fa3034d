import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import CausalTransformer, _lib
m = CausalTransformer()
e = torch.randn(135, 64, dtype=torch.float64).cuda() * 0.05
lib = _lib.load()
for rep in range(3):
    m.prefill_device(embeddings=e)
torch.cuda.synchronize()
# one forward; each tf_block launch overwrites the marks, so read after the whole forward = last layer
buf = (ctypes.c_ulonglong * (1024 * 16))()
lib.auras_tf_debug_times(buf, 1024 * 16)
T = np.array(buf[:135 * 16], dtype=np.int64).reshape(135, 16); t = T[:, :9]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
print("launch skew (start of CTAs) us: min %.2f max %.2f" % (rel[:, 0].min(), rel[:, 0].max()))
ph = np.diff(t, axis=1) / 1000.0
names = ["load", "attn", "merge", "wo", "ln2", "w1", "w2", "qkv/lnf"]
for i, nme in enumerate(names):
    print(f"{nme:8s} mean {ph[:, i].mean():6.2f} max {ph[:, i].max():6.2f} us  (row134 {ph[134, i]:.2f})")
print("CTA total mean %.2f max %.2f; kernel span %.2f" % ((t[:, 8]-t[:, 0]).mean()/1e3, (t[:, 8]-t[:, 0]).max()/1e3, (t[:, 8].max()-t0)/1e3))
