import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2509_09560_b200 import diffusion as D, _lib
cfg = D.PRESETS["vit"]
w = D.init_weights(cfg, 0, device="cpu")
model = D.DeviceModel(cfg, w, "bf16")
enc = D.ViTEncoder(model, 2)
lib = _lib.load()
st = torch.cuda.current_stream()
enc.img.copy_(torch.from_numpy(np.random.default_rng(3).integers(0, 256, (2, 3, 224, 224), dtype=np.uint8)))
_lib.check(lib.auras_image_to_nhwc(enc.img.data_ptr(), 2, 3, 224, 224, enc.x0.data_ptr(), 8, model.dt, st.cuda_stream), "i")
torch.cuda.synchronize(); print("nhwc ok")
import types
for gi, gname in enumerate(enc.GROUPS):
    items = enc.groups[gname]
    for j, item in enumerate(items):
        sub = types.SimpleNamespace()
        enc.groups[gname] = [item]
        try:
            if item[0] == "conv":
                op = item[1]
                print(gname, j, "conv M", op.M, "Cin", op.Cin, "Kp", op.Kp, "W", op.W, "act", op.act, "res", bool(op.res), flush=True)
            else:
                print(gname, j, item[0], flush=True)
            enc.groups[gname] = [item]
            if gi == 0 and j > 0:
                pass
            lo = gi
            # run just this item (skip image conversion by running with gi>0 trick)
            if item[0] == "conv":
                _lib.check(lib.auras_conv(_lib.C.byref(item[1]), model.dt, 2, None, 0, enc.scratch.data_ptr(), enc.scratch.numel(), st.cuda_stream), "conv")
            else:
                save = enc.GROUPS
                enc.GROUPS = ("x",) + tuple(save)
                enc.groups["x"] = []
                enc.run(gi + 1, gi + 2, st)
                enc.GROUPS = save
            torch.cuda.synchronize()
        except Exception as e:
            print("FAIL", gname, j, item[0], e); raise
        finally:
            enc.groups[gname] = items
    if gi >= 1: break
print("feat", enc.feat[:, :4])
