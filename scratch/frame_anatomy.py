import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=16)
rec = {}
orig_perceive = D.DPSession.perceive
orig_publish = D.DPSession.publish
orig_generate = D.DPSession.generate
def ev(stream):
    e = torch.cuda.Event(enable_timing=True); e.record(stream); return e
def perceive(self, lane, lo, hi):
    rec.setdefault("p0", []).append(ev(self.p)); rec.setdefault("hp0", []).append(time.perf_counter())
    orig_perceive(self, lane, lo, hi)
def publish(self, lane, frame, slot, version):
    orig_publish(self, lane, frame, slot, version)
    rec.setdefault("p1", []).append(ev(self.p)); rec.setdefault("hp1", []).append(time.perf_counter())
def generate(self, batch):
    rec.setdefault("g0", []).append(ev(self.g)); rec.setdefault("hg0", []).append(time.perf_counter())
    orig_generate(self, batch)
    rec.setdefault("g1", []).append(ev(self.g)); rec.setdefault("hg1", []).append(time.perf_counter())
D.DPSession.perceive, D.DPSession.publish, D.DPSession.generate = perceive, publish, generate
for il in ("1", "0"):
    os.environ["AURAS_INTERLEAVE_PG"] = il
    rec.clear()
    host = []
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8), pol, None, 40, clock="device",
                        frame_hook=lambda t, d, e: host.append(time.perf_counter()))
    torch.cuda.synchronize()
    base = rec["p0"][0]
    f = lambda k: np.array([base.elapsed_time(e) for e in rec[k]])
    p0, p1, g0, g1 = f("p0"), f("p1"), f("g0"), f("g1")
    n = min(len(p0), len(g0))
    print(f"interleave={il}: host frame ms {np.median(np.diff(host)[10:])*1e3:.2f}; perception span {np.median((p1-p0)[10:]):.2f} ms; "
          f"gen span {np.median((g1-g0)[10:]):.2f} ms; gen gap (g0[t+1]-g1[t]) {np.median((g0[11:]-g1[10:-1])):.2f} ms")
    print("  host: perceive->publish enqueue", np.median((np.array(rec['hp1'])-np.array(rec['hp0']))[10:])*1e3, "ms; generate enqueue", np.median((np.array(rec['hg1'])-np.array(rec['hg0']))[10:])*1e3, "ms")
    ft = res.frame_times; ends = np.array([ft["end"][i] for i in range(40)])
    print("  device frame ms", np.round(np.diff(ends)[10:20]*1e3, 2).tolist())
