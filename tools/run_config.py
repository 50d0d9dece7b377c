"""Time one BASELINE config on the GPU: `python tools/run_config.py C3 if4 [steps] [n]`.
Prints device ms per time step and grid-point-steps/s (second run, plan warm)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
key, scheme = sys.argv[1], sys.argv[2]
w = W.CONFIGS[key]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else w.steps
if len(sys.argv) > 4:
    w = w.scaled(int(sys.argv[4]), steps)
t0 = time.perf_counter()
x0 = W.initial_state_device(w)
prob = W.build_problem(w)
if w.boundary == "periodic":
    from paper_2403_02816_b200.spectral import fft_dev
    x0 = fft_dev(x0)
t_setup = time.perf_counter() - t0
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
print(json.dumps({"first_run_ms_per_step": 1e3 * r.device_seconds / steps}), flush=True)
if w.points < 2 ** 29:
    r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
print(json.dumps({"config": key, "scheme": scheme, "grid": list(w.extents), "steps": steps,
                  "ms_per_step": 1e3 * r.device_seconds / steps,
                  "gp_steps_per_s": w.points * steps / r.device_seconds, "diverged": r.diverged,
                  "setup_s": t_setup, "max_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
