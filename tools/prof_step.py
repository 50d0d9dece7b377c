"""Short C1 workload run for ncu (launch lists / full captures):
`python tools/prof_step.py [scheme] [time_steps]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

scheme = sys.argv[1] if len(sys.argv) > 1 else "if4"
key = sys.argv[3] if len(sys.argv) > 3 else "C1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = W.CONFIGS[key]
prob = W.build_problem(w)
x0 = torch.from_numpy(W.state_for_problem(w, W.initial_state(w))).cuda()
P.integrate(prob, scheme, (x0,), w.tau * steps, steps)  # warm: plans, graphs, workspaces
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
torch.cuda.synchronize()
print("ok", r.diverged, r.device_seconds / steps * 1e3, "ms/step")
