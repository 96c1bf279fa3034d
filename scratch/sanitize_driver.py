"""Minimal device work for compute-sanitizer runs: the ring stress kernel and one
cluster-kernel denoise launch (tiny, then pusht S=8), each checked for finiteness."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
os.environ.setdefault("AURAS_MEGA_KERNEL", "cluster")
from paper_2509_09560_b200 import _lib
what = sys.argv[1] if len(sys.argv) > 1 else "all"
lib = _lib.load()
if what in ("all", "ring"):
    counts = (ctypes.c_ulonglong * 8)()
    _lib.check(lib.auras_ring_stress(2, 256, 200, 2, counts), "ring_stress")
    print("ring counts", list(counts))
if what in ("all", "tiny", "pusht"):
    from dp_harness import norm_err, run_denoise_launch
    for cfg, S in (("tiny", 4), ("pusht", 8)):
        if what not in ("all", cfg):
            continue
        got, want, x0, kernel = run_denoise_launch(cfg, S)
        print(cfg, "S", S, "kernel", kernel, "err", norm_err(got, want), "finite", np.isfinite(got).all())
