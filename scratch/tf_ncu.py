import torch
from paper_2509_09560_b200 import CausalTransformer
m = CausalTransformer(); e = torch.randn(135, 64, dtype=torch.float64).cuda()
for _ in range(2):
    m.prefill_device(embeddings=e)
torch.cuda.synchronize()
