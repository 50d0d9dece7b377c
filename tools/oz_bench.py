"""Event-timed INT8-emulated mu-mode products on workload shapes (slicing +
GEMM, as the plans call them).  `python tools/oz_bench.py` -> one JSON line
per case.  For kernel A/B runs on one box build variants with
`python tools/oz_bench.py --build-variant NAME CSRC_DIR` and run with
CGL_LIB_OVERRIDE=paper_2403_02816_b200/_lib/NAME.so."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 3 and sys.argv[1] == "--build-variant":
    from paper_2403_02816_b200 import _build
    out = os.path.join(_build.LIB_DIR, sys.argv[2] + ".so")
    print(_build.build(force=True, csrc=sys.argv[3], out=out))
    sys.exit(0)

import torch  # noqa: E402

from paper_2403_02816_b200 import ozaki, workloads as W  # noqa: E402

CASES = [("C1", (512, 512), 0, 4), ("C1", (512, 512), 1, 4), ("C4", (1024, 1024, 128), 0, 1),
         ("C4", (128, 1024, 1024), 1, 1), ("C4", (128, 1024, 1024), 2, 1)]
reps = 30
for key, shape, axis, nf in CASES:
    w = W.CONFIGS[key]
    prob = W.build_problem(w)
    prob.operator.prepare(w.tau, (1,))
    fac = prob.operator.sliced_factors(1)[0]
    g = torch.Generator(device="cuda").manual_seed(1)
    ins = [torch.randn(shape, dtype=torch.complex128, device="cuda", generator=g) for _ in range(nf)]
    outs = [torch.empty_like(x) for x in ins]
    ws = ozaki.Workspace()
    for _ in range(3):
        ozaki.mode_product_oz(ins, [fac] * nf, outs, axis, ws)
    # replay a captured graph so the small C1 products are not host-launch bound
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            ozaki.mode_product_oz(ins, [fac] * nf, outs, axis, ws)
    torch.cuda.current_stream().wait_stream(s)
    graph.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps

    # the data slicing alone (same call the product makes first), captured the same way
    from paper_2403_02816_b200 import _lib
    lib = _lib.load()
    n = shape[axis]
    P = 1
    for d in shape[:axis]:
        P *= d
    Q = 1
    for d in shape[axis + 1:]:
        Q *= d
    bufs = [v for k, v in ws.bufs.items()]

    def slice_only():
        if Q > 1 and P == 1:
            _lib.check(lib.cgl_oz_slice_multi(_lib.stream(), ozaki.S, nf, _lib.ptr_array(ins), 1, Q, Q, n, 1, 0, 0,
                                              _lib.ptr_array([b[0] for b in bufs[:nf]]), 0,
                                              _lib.ptr_array([b[1] for b in bufs[:nf]]), 0), "slice")
        elif Q == 1:
            _lib.check(lib.cgl_oz_slice_multi(_lib.stream(), ozaki.S, nf, _lib.ptr_array(ins), n, 1, P, n, 1, 0, 0,
                                              _lib.ptr_array([b[0] for b in bufs[:nf]]), 0,
                                              _lib.ptr_array([b[1] for b in bufs[:nf]]), 0), "slice")
    us_slice = None
    if not (Q > 1 and P > 1):
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g2, stream=s):
                slice_only()
        torch.cuda.current_stream().wait_stream(s)
        g2.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            g2.replay()
        e1.record()
        torch.cuda.synchronize()
        us_slice = round(e0.elapsed_time(e1) * 1e3 / reps, 2)
    print(json.dumps({"case": key, "shape": shape, "axis": axis, "fields": nf, "us_per_product": round(us, 2),
                      "us_slicing": us_slice, "lib": os.environ.get("CGL_LIB_OVERRIDE", "default")}), flush=True)
