"""INT8 tensor-core fraction of the emulated mu-mode product at every FD config:
the axis-0 product of the step plans (ozgemm_persistent_kernel, data pre-sliced as in the step), executed
int8 MACs (zero blocks counted out) per launch over the launch time, against the measured tcgen05 kind::i8
issue rate (tools/mma_rate.cu) and against 2 x the measured bf16 rate; FP64-equivalent TFLOP/s alongside.

    python tools/oz_fraction.py [C1 C2 C4]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2403_02816_b200 import workloads as W  # noqa: E402

for key in (sys.argv[1:] or ["C1", "C2", "C4"]):
    w = W.CONFIGS[key]
    fields = 2
    if key == "C4":
        # the 1024^3 axis-0 product runs in column chunks of <= 2 GiB of slices per field; one chunk here:
        # the same (1024 x 1024) factor on 65536 of the 2^20 columns
        import dataclasses
        w = dataclasses.replace(w, extents=(1024, 64, 1024))
    r = bench.gemm_roofline(torch, w, scheme_fields=fields)
    n = w.extents[0]
    flops = 8.0 * n * w.points * fields          # FP64-equivalent flop of the product
    r["config"] = key
    r["fields"] = fields
    r["fp64_equiv_tflops"] = flops / (r["per_launch_ms"] * 1e-3) / 1e12
    r["bytes_per_point_gemm"] = None
    print(json.dumps(r), flush=True)
    torch.cuda.empty_cache()
