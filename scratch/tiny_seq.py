import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2509_09560_b200 import run_sequential
from paper_2509_09560_b200 import diffusion as D
w = D.init_weights(D.PRESETS["tiny"], 0, device="cpu")
pol = D.make_diffusion_policy("tiny", dtype="bf16", weights=w)
res = run_sequential(pol, None, int(sys.argv[1]) if len(sys.argv) > 1 else 4)
print("actions", len(res.actions), res.actions[0].values if res.actions else None)
