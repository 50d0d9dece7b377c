"""Per-launch timing of the batched DMMA mode product on workload shapes.
`python tools/gemm_bench.py` -> one JSON line per case (TFLOP/s algorithmic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_02816_b200 import _lib  # noqa: E402

lib = _lib.load()
CASES = [((512, 512), 0, 4), ((512, 512), 1, 4), ((512, 512), 0, 2), ((512, 512), 1, 2),
         ((128, 128), 0, 1), ((128, 128), 1, 1), ((256, 256, 256), 0, 1), ((256, 256, 256), 1, 1),
         ((256, 256, 256), 2, 1)]
if len(sys.argv) > 1:
    CASES = [CASES[int(i)] for i in sys.argv[1].split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
for shape, axis, nf in CASES:
    n = shape[axis]
    mats = [torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g) for _ in range(nf)]
    mts = [m.t().contiguous() for m in mats]
    ins = [torch.randn(shape, dtype=torch.complex128, device="cuda", generator=g) for _ in range(nf)]
    outs = [torch.empty_like(x) for x in ins]

    def launch():
        rc = lib.cgl_mode_product_batch(_lib.stream(), len(shape), _lib.i64_array(shape), axis, nf,
                                        _lib.ptr_array(mats), _lib.ptr_array(mts), n, _lib.ptr_array(ins),
                                        _lib.ptr_array(outs), 1.0, None, 0.0, None, 0)
        _lib.check(rc, "mode_product_batch")
    for _ in range(3):
        launch()
    # correctness vs torch (cuBLAS zgemm) on the first field
    want = torch.movedim(torch.tensordot(mats[0], ins[0], dims=([1], [axis])), 0, axis)
    err = ((outs[0] - want).abs().max() / want.abs().max()).item()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / reps
    pts = 1
    for s in shape:
        pts *= s
    fl = 8.0 * n * pts * nf
    print(json.dumps({"shape": shape, "axis": axis, "fields": nf, "us": dt * 1e6, "tflops": fl / dt / 1e12,
                      "rel_err_vs_cublas": err, "mode": os.environ.get("CGL_ZGEMM_4M", "0")}), flush=True)
