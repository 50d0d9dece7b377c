"""Achieved parity against the reference's recorded outputs (tests/golden):
relative L2 of every BASELINE-config fixture and the full-size C1 runs, for the
default plans (if4 in the "quad" form) and (if4) the reference-form plan (CGL_IF4_FORM=ref).
`python tools/parity_report.py` -> one line per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from conftest import GOLDEN, rel_l2  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

arrays = np.load(os.path.join(GOLDEN, "configs.npz"))
meta = {m["tag"]: m for m in json.load(open(os.path.join(GOLDEN, "configs.json")))}


def run(tag):
    m = meta[tag]
    w = W.CONFIGS[m["workload"].split("-")[0]]
    if "@" in m["workload"]:
        w = w.scaled(m["extents"][0], m["steps"])
    x0 = W.state_for_problem(w, W.initial_state(w))
    return P.integrate(W.build_problem(w), m["scheme"], (x0,), w.t_final, w.steps)


cases = ["C0_strang", "C1s64_if4", "C1s64_rk4", "C2s24_split4", "C3s32_if4", "C3s32_strang", "C4s24_if4",
         "C1_if4", "C1_strang", "C1_rk4"]
for form in ("quad", "ref"):
    os.environ["CGL_IF4_FORM"] = form
    for tag in cases:
        if form == "ref" and "if4" not in tag:
            continue
        want = arrays[f"{tag}_out"] if f"{tag}_out" in arrays else np.load(os.path.join(GOLDEN, f"{tag}_out.npy"))
        r = run(tag)
        fin = np.isfinite(want)
        err = rel_l2(r.fields[0][fin], want[fin]) if fin.any() else 0.0
        print(json.dumps({"case": tag, "if4_form": form, "rel_l2": err,
                          "diverged": r.diverged, "diverged_at": r.diverged_at}), flush=True)

# Full-size runs from the real reference kept as strided samples + checksums
# (tests/golden/make_golden_c2_full.py, make_golden_c3_steps.py).
os.environ["CGL_IF4_FORM"] = "quad"
sampled = []
p2 = os.path.join(GOLDEN, "C2_full_split4.npz")
if os.path.exists(p2):
    g = np.load(p2)
    sampled.append(("C2_full_split4", "C2", "split4", json.loads(str(g["meta"])), g["sample"], g["norm2"]))
p3 = os.path.join(GOLDEN, "C3_steps.npz")
if os.path.exists(p3):
    g = np.load(p3)
    for m in json.loads(str(g["meta"])):
        s = m["scheme"]
        sampled.append((f"C3_full_{s}_{m['steps']}steps", "C3", s, m, g[f"{s}_sample"], g[f"{s}_norm2"]))
for tag, key, scheme, m, want, norm2 in sampled:
    w = W.CONFIGS[key]
    x0 = W.state_for_problem(w, W.initial_state(w))
    r = P.integrate(W.build_problem(w), scheme, (x0,), w.tau * m["steps"], m["steps"])
    out = r.fields[0]
    got = out.reshape(-1, order="F")[m["offset"]::m["stride"]]
    print(json.dumps({"case": tag, "if4_form": "quad", "rel_l2_sample": rel_l2(got, want),
                      "rel_norm2": abs(float(np.vdot(out, out).real) - float(norm2)) / float(norm2),
                      "sample_points": int(want.size), "diverged": r.diverged,
                      "diverged_at": r.diverged_at}), flush=True)
    del out, r, x0
