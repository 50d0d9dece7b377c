"""Final state of a short run as .npy (bit-level A/B of kernel variants):
`python tools/state_dump.py C1 if4 60 out.npy` (CGL_LIB_OVERRIDE selects the library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

key, scheme, steps, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
w = W.CONFIGS[key]
prob = W.build_problem(w)
x0 = torch.from_numpy(W.state_for_problem(w, W.initial_state(w))).cuda()
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
f = r.fields[0]
np.save(out, f.cpu().numpy() if torch.is_tensor(f) else np.asarray(f))
print(key, scheme, steps, "diverged" if r.diverged else "ok")
