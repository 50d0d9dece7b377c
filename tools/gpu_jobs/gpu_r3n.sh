timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_experiments.py -m gpu -x -q > gpurun_out/n3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n3_pytest.log
tail -n 6 gpurun_out/n3_pytest.log
for v in 1 0 1 0; do echo "CGL_T2D_STEPS=$v"; CGL_T2D_STEPS=$v timeout 300 python tools/prof_step.py strang 200 C0; done
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2403_02816_b200 as P
from paper_2403_02816_b200 import workloads as W
w = W.CONFIGS["C0"]
outs = {}
for v in ("1", "0"):
    os.environ["CGL_T2D_STEPS"] = v
    x0 = torch.from_numpy(W.state_for_problem(w, W.initial_state(w))).cuda()
    r = P.integrate(W.build_problem(w), "strang", (x0,), w.t_final, w.steps)
    outs[v] = r.fields[0].clone()
print("bit-identical multi-step vs one launch per step:", bool(torch.equal(outs["1"], outs["0"])))
PY
