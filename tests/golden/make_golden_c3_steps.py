"""Full-grid C3 fixtures from the REAL reference (builder container only).

C3 = 3D periodic cubic CGL, Fourier pseudospectral on 512^3, tau = 0.01.  The
reference's 100-step runs take hours on pocketfft, so the fixture runs STEPS
(default 2) full-grid steps of if4 (Lawson-RK4) and strang from the config's
seeded u0 — the same per-step code at the full 512^3 size, which the 32^3
fixtures in configs.npz cannot exercise (cuFFT plan sizes, table indexing,
1/N folding).  Kept per scheme, as in make_golden_c2_full.py: a strided sample
of the final coefficient field (x1-fastest flattening), its squared L2 norm
and sum, and the divergence fields.
`python tests/golden/make_golden_c3_steps.py [steps]` -> tests/golden/C3_steps.npz
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
from cglsolve import spectral as rspec  # noqa: E402

import cgl_oracle as O  # noqa: E402
from make_golden_c2_full import OFFSET, STRIDE, sample  # noqa: E402


def main():
    from paper_2403_02816_b200 import workloads as W
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    w = W.CONFIGS["C3"]
    u0 = W.initial_state(w)
    p = cglsolve.CglParameters(**{k: getattr(w.params, k) for k in O.Params.NAMES})
    spec = rflows.NonlinearSpec(w.kind, p)
    grid = rspec.FourierGrid(w.extents, (w.interval,) * len(w.extents))
    prob = rint.Problem(rops.build_periodic_operator(grid, p), spec)
    x0 = rspec.dft_forward(u0)
    del u0
    arrays, metas = {}, []
    for scheme in ("strang", "if4"):
        t0 = time.perf_counter()
        res = rint.integrate(prob, scheme, (x0,), w.tau * steps, steps)
        out = res.fields[0]
        meta = dict(workload=w.name, scheme=scheme, extents=list(w.extents), steps=steps, tau=w.tau,
                    diverged=bool(res.diverged), diverged_at=int(res.diverged_at), reason=str(res.reason),
                    ref_seconds=res.seconds, wall=time.perf_counter() - t0, stride=STRIDE, offset=OFFSET)
        print(json.dumps(meta), flush=True)
        arrays[f"{scheme}_sample"] = sample(out)
        arrays[f"{scheme}_norm2"] = np.array(np.vdot(out, out).real)
        arrays[f"{scheme}_total"] = np.array(out.sum())
        metas.append(meta)
        del out, res
    np.savez_compressed(os.path.join(HERE, "C3_steps.npz"), meta=np.array(json.dumps(metas)), **arrays)


if __name__ == "__main__":
    main()
