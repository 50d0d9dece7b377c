"""C1 (512^2) rk4 / rk2 at a stable step size: device ms per time step (graph-captured BandedRKPlan)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

for scheme in ("rk4", "rk2"):
    w = dataclasses.replace(W.CONFIGS["C1"], tau=0.001)
    prob = W.build_problem(w)
    x0 = W.state_for_problem(w, W.initial_state_device(w))
    P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    print(scheme, "diverged", r.diverged, "ms/step", 1e3 * r.device_seconds / w.steps)
