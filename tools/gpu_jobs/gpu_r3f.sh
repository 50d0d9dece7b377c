cat > /tmp/san_fft.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2403_02816_b200 import _lib, fftpass
def rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.empty(shape, dtype=torch.complex128, device="cuda"); x.real.normal_(generator=g); x.imag.normal_(generator=g); return x
nl = _lib.Nonlinear(); nl.alpha3, nl.beta3, nl.kind = -1.0, 0.7, 0
# contiguous passes with pencil-level barriers (L = 512: named barriers; 128/64: warp barriers), strided passes, r32 G pass
for shape in [(16, 16, 512), (16, 32, 128), (512, 16, 16), (16, 512, 16), (64, 16, 64)]:
    x = rand(shape, 1)
    y = fftpass.fftn(x); z = fftpass.fftn(y, inverse=True)
    err = float((z / x.numel() - x).abs().max())
    assert err < 1e-12, (shape, err)
    for axis in (0, len(shape) - 1):
        out = torch.empty_like(x)
        fftpass.axis_pass(x, out, axis, program="g", ops=fftpass.make_ops(nl=nl, scale=0.05))
torch.cuda.synchronize()
# stage programs between transforms (B1..B4, STR_MID) on a small 3D grid through the plan
import paper_2403_02816_b200 as P
from paper_2403_02816_b200 import workloads as W
for scheme in ("if4", "strang"):
    w = W.CONFIGS["C3"].scaled(32, 3)
    prob = W.build_problem(w)
    x0 = W.state_for_problem(w, W.initial_state_device(w))
    r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    assert not r.diverged
# banded RK stage
w = W.CONFIGS["C1"].scaled(64, 4)
r = P.integrate(W.build_problem(w), "rk4", (W.state_for_problem(w, W.initial_state_device(w)),), 4e-4, 4)
assert not r.diverged
print("sanitizer workload ok")
PY
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san_fft.py > gpurun_out/f3_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/f3_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san_fft.py > gpurun_out/f3_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/f3_racecheck.log
tail -n 6 gpurun_out/f3_memcheck.log; tail -n 12 gpurun_out/f3_racecheck.log
