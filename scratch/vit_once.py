import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["vit"]
w = D.init_weights(cfg, 0, device="cpu")
model = D.DeviceModel(cfg, w, "bf16")
enc = D.ViTEncoder(model, 1)
st = torch.cuda.current_stream()
enc.run(0, 5, st); torch.cuda.synchronize()
enc.run(0, 5, st); torch.cuda.synchronize()
