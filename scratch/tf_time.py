import os, sys, json, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import CausalTransformer
m = CausalTransformer()
e = torch.randn(135, 64, dtype=torch.float64).cuda() * 0.05
for _ in range(3):
    m.prefill_device(embeddings=e)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        for _ in range(20):
            h, _ = m.prefill_device(embeddings=e)
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); 
for _ in range(5): g.replay()
b.record(); b.synchronize()
print(os.environ.get("AURAS_LIB", "default"), "merged prefill (135 rows) us:", a.elapsed_time(b) / 100 * 1e3)
