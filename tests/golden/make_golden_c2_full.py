"""Full-size C2 fixture from the REAL reference (run in the builder container,
where /root/reference exists; the fixture travels, the reference does not).

C2 = 3D cubic-quintic CGL, 256^3 Neumann FD, split4 (the reference's 4th-order
splitting, integrators.py:161-190), tau = 0.01, 100 steps.  The full output is
268 MB, so the fixture keeps what a size-independent comparison needs:
  * a fixed strided sample of the flattened (x1-fastest) final field
    (every STRIDE-th point from OFFSET; a stride coprime to 256 so the sample
    visits every x1/x2/x3 residue),
  * the global squared L2 norm and the sum of the field (a checksum that sees
    every point),
  * diverged / diverged_at / reason.
`python tests/golden/make_golden_c2_full.py [steps]` -> tests/golden/C2_full_split4.npz
(steps < 100 only for timing the generator; the committed file is the full run).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, REPO)

import cglsolve  # noqa: E402  (the reference)
from cglsolve import flows as rflows  # noqa: E402
from cglsolve import integrators as rint  # noqa: E402
from cglsolve import operators as rops  # noqa: E402

import cgl_oracle as O  # noqa: E402

STRIDE = 4099
OFFSET = 17


def sample(x):
    return np.ascontiguousarray(x.reshape(-1, order="F")[OFFSET::STRIDE])


def main():
    from paper_2403_02816_b200 import workloads as W
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else None
    w = W.CONFIGS["C2"]
    n_steps = steps or w.steps
    t_final = w.tau * n_steps
    u0 = W.initial_state(w)
    p = cglsolve.CglParameters(**{k: getattr(w.params, k) for k in O.Params.NAMES})
    spec = rflows.NonlinearSpec(w.kind, p)
    a, b = w.interval
    d = len(w.extents)
    mats = [p.diffusion * O.FD_BUILDERS[w.boundary](n, b - a) + (p.alpha2 / d) * np.eye(n) for n in w.extents]
    prob = rint.Problem(rops.KroneckerOperator(mats), spec)
    t0 = time.perf_counter()
    res = rint.integrate(prob, "split4", (u0,), t_final, n_steps)
    dt = time.perf_counter() - t0
    out = res.fields[0]
    meta = dict(workload=w.name, scheme="split4", extents=list(w.extents), steps=n_steps, tau=w.tau,
                diverged=bool(res.diverged), diverged_at=int(res.diverged_at), reason=str(res.reason),
                ref_seconds=res.seconds, wall=dt, stride=STRIDE, offset=OFFSET,
                boundary=w.boundary)
    print(json.dumps(meta))
    if steps is None:
        np.savez_compressed(os.path.join(HERE, "C2_full_split4.npz"), sample=sample(out),
                            norm2=np.array(np.vdot(out, out).real), total=np.array(out.sum()),
                            meta=np.array(json.dumps(meta)))


if __name__ == "__main__":
    main()
