"""Full-length runs against the REAL reference (tests/golden/full_<C>_<n>.npz,
made by tests/golden/make_golden_full.py from `cglsolve.integrate`,
integrators.py:241-282).

BASELINE's bar is relative L2 <= 1e-10 "after the full run".  The fixtures
hold, per scheme, a strided sample of the final field, its squared L2 norm
and sum (checksums over every point), and the LOW-AMPLITUDE region: points
where |u_ref| < 1e-6 max|u_ref| and < 1e-3 max|u_ref|.  The INT8-emulated
mu-mode products (ozaki.py) round relative to row-max x column-max, so the
error there is bounded separately: max |u - u_ref| over the band, relative to
the band's largest |u_ref| (`band_rel`), and relative to the global peak
(`band_abs`, the FP64-GEMM error model: a few ulp of the peak).

C3 (512^3 Fourier) and C4 (FD Dirichlet) run at their full step counts; C4's
1024^3 grid needs ~210 GB of host RAM for the reference, so its full 50 steps
are pinned at 64^3 and 256^3 on the identical code path (the
reference takes 26 min at 256^3 and would take ~3.4 h at 512^3, where its
first 16 steps are pinned: steps_C4_512.npz, 64 min of reference time).
"""

import glob
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

STRIDE, OFFSET = 4099, 17
RESULTS = os.environ.get("CGL_FULLRUN_LOG")  # optional JSON-lines record of the measured errors


def _cases():
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "full_*.npz")) + glob.glob(os.path.join(GOLDEN, "steps_*.npz"))):
        with np.load(path) as z:
            for m in json.loads(str(z["meta"])):
                out.append((os.path.basename(path), m["scheme"]))
    return out


@pytest.mark.parametrize("fname,scheme", _cases())
def test_full_run_against_reference(fname, scheme):
    import paper_2403_02816_b200 as P
    from paper_2403_02816_b200 import workloads as W
    z = np.load(os.path.join(GOLDEN, fname))
    meta = next(m for m in json.loads(str(z["meta"])) if m["scheme"] == scheme)
    base = W.CONFIGS[meta["config"]]
    n = meta["extents"][0]
    w = base if n == base.extents[0] else base.scaled(n)
    if fname.startswith("steps_"):   # the first meta["steps"] steps of the run (512^3 C4: ~8 min of reference per step)
        w = w.scaled(n, meta["steps"])
    assert list(w.extents) == meta["extents"] and meta["steps"] == w.steps and meta["tau"] == w.tau
    prob = W.build_problem(w)
    x0 = W.state_for_problem(w, W.initial_state_device(w))
    res = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    assert (res.diverged, res.diverged_at, res.reason) == (meta["diverged"], meta["diverged_at"], meta["reason"])
    u = res.fields[0]
    flat = u.permute(*reversed(range(u.ndim))).reshape(-1)   # x1-fastest flattening (F order)
    sample = flat[OFFSET::STRIDE].cpu().numpy()
    ref = z[f"{scheme}_sample"]
    norm2 = float(torch.vdot(flat, flat).real)
    # the sample's error against the field's RMS magnitude estimates the global
    # relative L2 (a strided sample can land entirely in near-zero regions, e.g.
    # C4's Gaussians in (-30, 30)^3, where a ratio to the sample's own norm
    # measures the low-amplitude error instead -- that is the `bands` check)
    rel_sample = float(np.linalg.norm(sample - ref) / np.sqrt(float(z[f"{scheme}_norm2"]) * ref.size / flat.numel()))
    rel_norm2 = abs(norm2 - float(z[f"{scheme}_norm2"])) / float(z[f"{scheme}_norm2"])
    total = complex(flat.sum())
    rel_total = abs(total - complex(z[f"{scheme}_total"])) / np.sqrt(flat.numel() * float(z[f"{scheme}_norm2"]))
    peak = float(z[f"{scheme}_peak"])
    bands = {}
    for band in ("lo6", "lo3"):
        idx = z[f"{scheme}_{band}_idx"]
        if idx.size == 0:
            continue
        got = flat[torch.from_numpy(idx).to(flat.device)].cpu().numpy()
        val = z[f"{scheme}_{band}_val"]
        err = float(np.max(np.abs(got - val)))
        bands[band] = {"count": int(z[f"{scheme}_{band}_count"]), "checked": int(idx.size),
                       "band_rel": err / float(np.max(np.abs(val))), "band_abs": err / peak}
    rec = dict(case=fname, scheme=scheme, extents=meta["extents"], steps=meta["steps"], rel_l2_sample=rel_sample,
               rel_norm2=rel_norm2, rel_total=rel_total, bands=bands, device_seconds=res.device_seconds)
    print(json.dumps(rec))
    if RESULTS:
        with open(RESULTS, "a") as f:
            f.write(json.dumps(rec) + "\n")
    assert rel_sample <= 1e-10
    assert rel_norm2 <= 2e-10
    assert rel_total <= 1e-10
    for band, b in bands.items():
        # the FP64 error model of the reference's own zgemm / pocketfft: a few
        # hundred ulp of the global peak after the full run
        assert b["band_abs"] <= 1e-12, (band, b)


def test_low_amplitude_error_model_int8_vs_dmma(monkeypatch):
    """The INT8-emulated products (ozaki.py) round relative to row-max x
    column-max; the DMMA products per element.  On C4 at 64^3 (Gaussians in
    (-30, 30)^3: 75% of the points are below 1e-6 of the peak) both engines
    meet the global bar after the full 50 steps; in the low band the emulated
    engine's error relative to the band's own scale is larger.  Recorded, and
    bounded: <= 1e-6 of the band scale and <= 1e-12 of the peak."""
    import paper_2403_02816_b200 as P
    from paper_2403_02816_b200 import workloads as W
    path = os.path.join(GOLDEN, "full_C4_64.npz")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    z = np.load(path)
    w = W.CONFIGS["C4"].scaled(64)
    idx = torch.from_numpy(z["if4_lo6_idx"])
    val = z["if4_lo6_val"]
    out = {}
    for engine in ("oz", "dmma"):
        monkeypatch.setenv("CGL_GEMM", engine)
        prob = W.build_problem(w)
        r = P.integrate(prob, "if4", (W.initial_state_device(w),), w.t_final, w.steps)
        flat = r.fields[0].permute(2, 1, 0).reshape(-1)
        got = flat[idx.to(flat.device)].cpu().numpy()
        out[engine] = float(np.max(np.abs(got - val)) / np.max(np.abs(val)))
    print(json.dumps({"lo6_band_rel": out}))
    if RESULTS:
        with open(RESULTS, "a") as f:
            f.write(json.dumps({"case": "low_amplitude_C4_64", "lo6_band_rel": out}) + "\n")
    assert out["oz"] <= 1e-6 and out["dmma"] <= 1e-6
