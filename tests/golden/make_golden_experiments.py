"""Golden fixtures for the harness layer (experiments / CLI callers).

Runs the reference package `cglsolve` (/root/reference/pkg/src, imported
in the build container only) on the desk-scale presets with short runs and
records: every preset's initial state, run_preset summaries, a
convergence study (exact plane-wave reference) and a stability sweep.
Writes tests/golden/experiments.npz + experiments.json.

    python tests/golden/make_golden_experiments.py
"""

import json
import os
import sys
import time
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import cglsolve.experiments as E  # noqa: E402  (the reference)

arrays, meta = {}, {"presets": {}, "runs": {}, "study": None, "sweep": None}
t0 = time.time()
for name in E.available_presets():
    cfg = E.make_preset(name)
    ics = E.initial_state(cfg)
    for k, u in enumerate(ics):
        arrays[f"ic_{name}_{k}"] = np.asarray(u)
    meta["presets"][name] = {"extents": list(cfg.extents), "ncomp": len(ics), "kind": cfg.kind,
                             "boundary": cfg.boundary, "t_final": cfg.t_final, "scheme": cfg.scheme,
                             "steps": cfg.steps}

# short runs of three presets (steps reduced so the reference finishes quickly)
for name, steps, t_final in (("plane-wave-1d", 40, None), ("cubic-2d-periodic", 40, 1.2),
                             ("cubic-2d-dirichlet", 30, 0.9)):
    cfg = E.make_preset(name)
    cfg = replace(cfg, steps=steps, **({"t_final": t_final} if t_final else {}))
    summary, phys = E.run_preset(cfg)
    summary.pop("seconds")
    summary.pop("snapshots")
    meta["runs"][name] = {"summary": summary, "steps": steps, "t_final": cfg.t_final}
    for k, u in enumerate(phys):
        arrays[f"run_{name}_{k}"] = np.asarray(u)

cfg = E.make_preset("plane-wave-1d")
rows, m = E.run_convergence_study(cfg, ["if4", "strang", "split4"], [14, 20, 28])
meta["study"] = {"rows": [{k: v for k, v in r.items() if k != "seconds"} for r in rows], "meta": m}

# long horizon: rk2 and if2 blow up (at different steps), strang survives
cfg = replace(E.make_preset("cubic-2d-dirichlet"), t_final=600.0)
table = E.stability_sweep(cfg, ["rk2", "if2", "strang"], [100, 200, 800])
meta["sweep_t_final"] = 600.0
meta["sweep"] = {s: [{k: v for k, v in o.items() if k != "seconds"} for o in outs] for s, outs in table.items()}

np.savez_compressed(os.path.join(HERE, "experiments.npz"), **arrays)
with open(os.path.join(HERE, "experiments.json"), "w") as fh:
    json.dump(meta, fh, indent=1, default=float)
print(f"wrote experiments fixtures ({len(arrays)} arrays) in {time.time() - t0:.1f} s")
