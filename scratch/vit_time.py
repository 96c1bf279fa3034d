import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["vit"]
w = D.init_weights(cfg, 0, device="cpu")
model = D.DeviceModel(cfg, w, "bf16")
for A in (1, 8):
    enc = D.ViTEncoder(model, A)
    st = torch.cuda.current_stream()
    for _ in range(3):
        enc.run(0, 5, st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        enc.run(0, 5, st)
    b.record(); b.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"ViT-B/16 A={A}: {ms:.3f} ms per forward, {35.1 * A / ms:.1f} TFLOP/s")
