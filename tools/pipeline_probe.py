import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2604_10377_b200 as fm
from paper_2604_10377_b200 import synth
cfg = synth.CONFIGS["cfg2"]
data = synth.make_batch(cfg)
t = {k: torch.from_numpy(v).cuda() for k, v in data.items()}
opts = fm.SolverOptions(compute_residual=False)
run = lambda: fm.pipeline_device(t["phi1"], t["mass1"], t["F1"], t["ev1"], t["phi2"], t["mass2"], t["F2"], t["ev2"], lam=cfg.lam, sigma=cfg.sigma, opts=opts)
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); e1.synchronize()
print("pipeline ms", e0.elapsed_time(e1) / 10)
