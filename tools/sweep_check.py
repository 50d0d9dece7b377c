import sys, numpy as np, json
sys.path.insert(0, "/root/repo")
import torch
from dataclasses import replace
from paper_2403_02816_b200 import experiments as X, integrate
arr = np.load("/root/repo/tests/golden/experiments.npz")
cfg = replace(X.make_preset("cubic-2d-dirichlet"), t_final=600.0)
prob = X.build_problem(cfg)
u_ref = arr["ic_cubic-2d-dirichlet_0"]
u_dev = X.initial_state(cfg)[0]
print("ic max diff", np.max(np.abs(u_ref - u_dev)), np.max(np.abs(u_ref)))
for name, u in (("reference IC", u_ref), ("device IC", u_dev)):
    for m in (100, 200, 800):
        r = integrate(prob, "if2", (torch.from_numpy(u).cuda(),), 600.0, m)
        print(name, m, r.diverged, r.diverged_at, r.reason)
