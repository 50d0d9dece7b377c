import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2403_02816_b200 as P
from paper_2403_02816_b200 import workloads as W
w = W.CONFIGS["C1"]
u0 = W.initial_state(w)
for s in sys.argv[1:]:
    try:
        r = P.integrate(W.build_problem(w), s, (u0,), w.t_final, w.steps)
        print(s, "ok", r.diverged, r.device_seconds)
    except Exception as e:
        print(s, "FAIL", repr(e)[:300])
