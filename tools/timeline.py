"""In-graph kernel timeline of one workload (profiling build, -DCGL_PROF).

    python tools/timeline.py [--build] [C1] [if4] [steps]

Builds `_lib/libcgl_prof.so` (with --build), runs the workload once warm,
then once more with every warp of the instrumented kernels recording its
start/end (globaltimer), and prints, for one steady-state time step, each
launch's span, the spread of its CTA start/end times and (persistent GEMM)
the per-role warp end times.  Unlike an ncu launch list this sees the
graph-replayed step as it runs: PDL overlap, warm L2, no serialisation.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_LIB = os.path.join(ROOT, "paper_2403_02816_b200", "_lib", "libcgl_prof.so")

args = [a for a in sys.argv[1:] if not a.startswith("--")]
if "--build" in sys.argv or not os.path.exists(PROF_LIB):
    from paper_2403_02816_b200 import _build
    _build.build(force=True, out=PROF_LIB, extra_flags=["-DCGL_PROF"])
os.environ["CGL_LIB_OVERRIDE"] = PROF_LIB

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import _lib, workloads as W  # noqa: E402

KID = {1: "slice_tile", 2: "ozgemm_persistent", 3: "stage", 4: "stage_slice", 5: "flag_advance", 6: "separable",
       7: "zgemm", 8: "ozgemm", 9: "rowexp", 10: "zmap", 11: "lincomb", 12: "pointwise"}

key = args[0] if args else "C1"
scheme = args[1] if len(args) > 1 else "if4"
steps = int(args[2]) if len(args) > 2 else 32
w = W.CONFIGS[key]
prob = W.build_problem(w)
x0 = W.initial_state_device(w)
if w.boundary == "periodic":
    from paper_2403_02816_b200.spectral import fft_dev
    x0 = fft_dev(x0)
lib = _lib.load()
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)  # warm: plans + graphs
cap = 1 << 22
rec = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
cnt = torch.zeros(256, dtype=torch.int64, device="cuda")  # per-SM counters
_lib.check(lib.cgl_prof_set(_lib.c_ptr(rec.data_ptr()), _lib.c_ptr(cnt.data_ptr()), cap), "cgl_prof_set")
torch.cuda.synchronize()
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
torch.cuda.synchronize()
per_sm = cap // 256
counts = np.minimum(cnt.cpu().numpy(), per_sm)
rv = rec.view(256, per_sm, 4).cpu().numpy()
a = np.concatenate([rv[sm, :counts[sm]] for sm in range(256)])
n = len(a)
t0, t1 = a[:, 0], a[:, 1]
kid = (a[:, 2] & 0xFFFFFFFF).astype(np.int64)
blk = (a[:, 2] >> 32).astype(np.int64)
warp = (a[:, 3] & 0xFFFFFFFF).astype(np.int64)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"tl_{key}_{scheme}{os.environ.get('TL_TAG', '')}.npz"), a=a)
print(f"# {key} {scheme}: {steps} steps, device {1e3 * r.device_seconds / steps:.4f} ms/step, {n} warp records")

# in-kernel marks (ids >= 100) are reported with the launch they fall in
MARKS = {101: "setup done", 110: "pro pdl passed", 111: "pro vb1", 112: "pro vb2", 113: "pro work done",
         102: "prologue+barrier done", 103: "issuer first data", 104: "issuer done", 105: "epilogue done", 106: "producers done", 107: "producer pdl passed", 109: "w0 init", 114: "list built", 115: "A copy issued", 108: "producer flag read",
         201: "pdl wait passed", 202: "stage computed", 203: "exponents known",
         301: "pdl wait passed", 302: "staged", 303: "cluster synced"}
MARKS_OF = {"ozgemm_persistent": (109, 101, 114, 115, 110, 111, 112, 113, 102, 107, 108, 103, 104, 105, 106), "stage_slice": (201, 202, 203),
            "slice_tile": (301, 302, 303, 201, 203)}
is_mark = kid >= 100
mk_t1, mk_kid = t1[is_mark], kid[is_mark]
t0, t1, kid, blk, warp = t0[~is_mark], t1[~is_mark], kid[~is_mark], blk[~is_mark], warp[~is_mark]

# group records into launches: per kernel id, the k-th record (by start
# time) of a given (block, warp) belongs to that kernel's k-th launch
launches = []
for k in np.unique(kid):
    idx = np.where(kid == k)[0]
    idx = idx[np.argsort(t0[idx], kind="stable")]
    seen, groups = {}, []
    for i in idx:
        c = seen.get((blk[i], warp[i]), 0)
        seen[(blk[i], warp[i])] = c + 1
        if c == len(groups):
            groups.append([])
        groups[c].append(i)
    launches += [(k, np.array(g)) for g in groups]
launches.sort(key=lambda L: t0[L[1]].min())

# one steady-state step: the launches between the (steps/2)-th and the next
# flag_advance (end-of-chunk) is too coarse; use the kernel sequence period
names = [KID[k] for k, _ in launches]
starts = np.array([t0[ix].min() for _, ix in launches])
ends = np.array([t1[ix].max() for _, ix in launches])
# period = number of launches per step (total / steps, ignoring prologue/epilogue kernels)
per = max(1, round((len(launches) - 2) / steps))
mid = len(launches) // 2
mid -= mid % per
lo = mid
hi = min(len(launches), lo + per)
base = starts[lo]
print(f"# launches per step ~{per}; step window {lo}..{hi - 1}; times in us from the window's first start")
print(f"{'kernel':20s} {'ctas':>5s} {'start':>7s} {'end':>7s} {'span':>6s} {'gap':>6s}  blk-start(min/med/max)  blk-end(min/med/max)")
prev_end = None
for j in range(lo, hi):
    k, ix = launches[j]
    b = blk[ix]
    ub = np.unique(b)
    bs = np.array([t0[ix][b == u].min() for u in ub])
    be = np.array([t1[ix][b == u].max() for u in ub])
    gap = (starts[j] - prev_end) / 1e3 if prev_end is not None else 0.0
    print(f"{KID[k]:20s} {len(ub):5d} {(starts[j] - base) / 1e3:7.2f} {(ends[j] - base) / 1e3:7.2f} "
          f"{(ends[j] - starts[j]) / 1e3:6.2f} {gap:6.2f}  "
          f"{(bs.min() - base) / 1e3:6.2f}/{(np.median(bs) - base) / 1e3:6.2f}/{(bs.max() - base) / 1e3:6.2f}  "
          f"{(be.min() - base) / 1e3:6.2f}/{(np.median(be) - base) / 1e3:6.2f}/{(be.max() - base) / 1e3:6.2f}")
    if KID[k] in MARKS_OF:
        inside = (mk_t1 >= starts[j]) & (mk_t1 <= ends[j])
        line = "   marks min/med/max:"
        for m in MARKS_OF[KID[k]]:
            nm = MARKS[m]
            e = mk_t1[inside & (mk_kid == m)]
            if len(e):
                line += f" | {nm} {(e.min() - base) / 1e3:.2f}/{(np.median(e) - base) / 1e3:.2f}/{(e.max() - base) / 1e3:.2f}"
        print(line)
    prev_end = ends[j]
period = np.median(starts[lo + per:len(starts) - per] - starts[lo:len(starts) - 2 * per]) if len(starts) > 3 * per else float("nan")
gaps = starts[1:] - np.maximum.accumulate(ends)[:-1]
big = np.where(gaps > 5e3)[0]
print(f"# median step period {period / 1e3:.2f} us; {len(big)} gaps > 5 us totalling {gaps[big].sum() / 1e3:.1f} us "
      f"over the run ({(starts[-1] - starts[0]) / 1e3:.1f} us): " + ", ".join(f"{gaps[i] / 1e3:.1f} before {names[i + 1]}#{i + 1}" for i in big[:12]))
print(f"# step window span {(ends[lo:hi].max() - starts[lo]) / 1e3:.2f} us; next step starts "
      f"{(starts[hi] - starts[lo]) / 1e3 if hi < len(starts) else float('nan'):.2f} us after")
