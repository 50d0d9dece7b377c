"""Benchmark of the CGL hot path on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
2D cubic CGL, 512x512 interior points, 2nd-order FD Dirichlet, complex128,
Lawson-RK4 (`if4`), tau = 0.005, 400 time steps, seeded u0 (workloads.C1).

One bench "step" = one full `integrate()` run of that workload (400 time
steps).  Metric = grid-point-steps/s = N_points * time_steps / second over
the stepping loop (the reference's own timing scope, integrators.py:258-281,
prepare excluded).
  value   device time (CUDA events) of the loop, state resident in HBM, L2
          flushed between bench steps (256 MiB write); max over ranks.
  e2e     the public API with HOST input/output (pinned host tensor in,
          numpy out): H2D + loop + D2H inside the timed region.
  roofline  the DMMA mu-mode-product GEMM (dominant kernel): algorithmic
          8*n flops per point per product, timed per launch with CUDA events
          on the C1 shapes, against the FP64 DMMA peak measured live by
          cgl_probe_dmma in the same process.
  cpu_baseline  the CPU oracle port (numpy/OpenBLAS, same algorithm as the
          reference) on a bounded sample of the same workload, rank 0, N=1.

--impl reference runs that CPU port instead (the reference is pure Python
+ numpy and cannot travel to the box; oracle/cgl_oracle.py restates it and
is pinned to the reference's own outputs by tests/test_oracle_golden.py).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FP64_PEAK_RECORDED = 37.06  # TFLOP/s, tools/fp64_peak.cu on this pool (profiles/fp64_peak_r01.txt)
METRIC = "grid-point-steps/s"
UNIT = "gp-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="C1")
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--no-extras", action="store_true", help="skip strang/rk4 side runs and the CPU sample")
    ap.add_argument("--cpu-sample-steps", type=int, default=24)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# CPU side (oracle port): the reference arm and the cpu_baseline leg
# ---------------------------------------------------------------------------

def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_run(w, scheme, max_steps):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cgl_oracle as O
    from paper_2403_02816_b200 import workloads as W
    from threadpoolctl import threadpool_limits
    p = O.Params(**{k: getattr(w.params, k) for k in O.Params.NAMES})
    u0 = W.initial_state(w)
    if w.boundary == "periodic":
        blocks = [O.FourierOp(O.symbol(w.extents, (w.interval,) * len(w.extents), p))]
        x0 = np.fft.fftn(u0)
    else:
        a, b = w.interval
        d = len(w.extents)
        blocks = [O.KronOp([p.diffusion * O.FD_BUILDERS[w.boundary](n, b - a) + (p.alpha2 / d) * np.eye(n)
                            for n in w.extents])]
        x0 = u0
    with threadpool_limits(limits=cpu_cores()):
        res = O.integrate(O.Prob(blocks, w.kind, p), scheme, (x0,), w.t_final, w.steps, max_steps=max_steps)
    done = res.diverged_at if res.diverged else min(w.steps, max_steps)
    return res.seconds, done


def reference_arm(args, w, scheme):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sample = max(1, args.cpu_sample_steps // 3)
    for _ in range(args.warmup):
        oracle_run(w, scheme, sample)
    tot_s, tot_steps = 0.0, 0
    for _ in range(args.steps):
        s, n = oracle_run(w, scheme, sample)
        tot_s += s
        tot_steps += n
    v = w.points * tot_steps / tot_s
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(w, scheme, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sample} of {w.steps} {scheme} time steps per bench step on {w.extents} "
                                   f"(oracle/cgl_oracle.py, numpy {np.__version__}, OpenBLAS {cores} threads)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(w, scheme, world):
    return {"workload": w.name, "grid": list(w.extents), "boundary": w.boundary, "scheme": scheme,
            "tau": w.tau, "time_steps": w.steps, "dtype": "complex128",
            "bench_step": f"one integrate() run = {w.steps} {scheme} time steps",
            "l2": "flushed (256 MiB write) between bench steps; within a run the state stays resident",
            "parallelism": f"replicas x{world}" if world > 1 else "single"}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(buf):
    buf.zero_()


def gemm_roofline(torch, w, scheme_fields=4):
    """Time the dominant kernel (batched DMMA mode product, C1 shapes) per
    launch with CUDA events; return achieved/peak TFLOP/s."""
    from paper_2403_02816_b200 import _lib, workloads as W
    lib = _lib.load()
    n1, n2 = w.extents
    prob = W.build_problem(w)
    prob.operator.prepare(w.tau, (1,))
    mats, mts = prob.operator.exp_factors(1)
    g = torch.Generator(device="cuda").manual_seed(0)
    ins = [torch.randn(w.extents, dtype=torch.complex128, device="cuda", generator=g) for _ in range(scheme_fields)]
    outs = [torch.empty_like(x) for x in ins]
    shape = _lib.i64_array(w.extents)
    res = {}
    for axis in (0, 1):
        def launch():
            # one launch = `scheme_fields` fields through mode `axis` (as in the if4 step)
            rc = lib.cgl_mode_product_batch(_lib.stream(), 2, shape, axis, scheme_fields,
                                            _lib.ptr_array([mats[axis]] * scheme_fields),
                                            _lib.ptr_array([mts[axis]] * scheme_fields), w.extents[axis],
                                            _lib.ptr_array(ins), _lib.ptr_array(outs), 1.0, None, 0.0, None, 0)
            _lib.check(rc, "cgl_mode_product_batch")
        for _ in range(3):
            launch()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3 / reps
        flops = 8.0 * w.extents[axis] * n1 * n2 * scheme_fields
        res[axis] = (flops, dt)
    # live FP64 DMMA peak
    stream = _lib.stream()
    lib.cgl_probe_dmma(stream, 256)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        e0.record()
        fl = lib.cgl_probe_dmma(stream, 4096)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, fl / (e0.elapsed_time(e1) / 1e3) / 1e12)
    flops = sum(f for f, _ in res.values())
    dt = sum(t for _, t in res.values())
    achieved = flops / dt / 1e12
    m3 = os.environ.get("CGL_ZGEMM_4M", "0") != "1"
    return {"bound": "tensor", "achieved": achieved, "peak": best, "unit": "TFLOP/s", "frac": achieved / best,
            "traffic": None,
            "kernel": "zgemm_kernel<64,64,32,4,4,2,3M> (DMMA.8x8x4, stream-K), 4-field batched mode products "
                      "of the if4 step (M=N=K=512 per field)",
            "complex_product": "3M (3 DMMA per complex MAC)" if m3 else "4M",
            "executed_dmma_frac": achieved * (0.75 if m3 else 1.0) / best,
            "per_launch_ms": {f"mode{a + 1}": 1e3 * t for a, (_, t) in res.items()},
            "algorithmic_flops_per_launch": {f"mode{a + 1}": f for a, (f, _) in res.items()},
            "peak_source": f"cgl_probe_dmma live in this run (recorded {FP64_PEAK_RECORDED} TFLOP/s, "
                           "tools/fp64_peak.cu); MEASURED_PEAKS.json has no FP64 figure"}


def gpu_arm(args, w, scheme):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2403_02816_b200 as P
    from paper_2403_02816_b200 import _lib, workloads as W
    lib = _lib.load()

    prob = W.build_problem(w)
    u0 = W.initial_state(w)
    x0_host = W.state_for_problem(w, u0)
    x0 = torch.from_numpy(np.ascontiguousarray(x0_host)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(args.warmup):
        r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    n_launch0 = lib.cgl_launch_count()
    replay0 = sum(fp.replayed_launches for fp in getattr(prob, "_plans", {}).values())
    dev_total = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
            dev_total += r.device_seconds
    launches = lib.cgl_launch_count() - n_launch0 + sum(
        fp.replayed_launches for fp in getattr(prob, "_plans", {}).values()) - replay0
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([dev_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_total = float(t.item())
    steps_done = (r.diverged_at if r.diverged else w.steps)
    value = world * w.points * steps_done * args.steps / dev_total

    # e2e through the public API with host buffers (pinned host tensor in, numpy out)
    x_pinned = torch.from_numpy(np.ascontiguousarray(x0_host)).pin_memory()
    P.integrate(prob, scheme, (x_pinned,), w.t_final, w.steps)
    e2e_total = 0.0
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = P.integrate(prob, scheme, (x_pinned,), w.t_final, w.steps)
        _ = r2.fields[0]  # numpy array on the host
        torch.cuda.synchronize()
        e2e_total += time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e = world * w.points * steps_done * args.steps / e2e_total

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(w, scheme, world),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16 * w.points,
                "d2h_bytes_per_step": 16 * w.points, "ms_per_step": 1e3 * e2e_total / args.steps},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "diverged": bool(r.diverged),
    }
    if rank == 0:
        try:
            line["roofline"] = gemm_roofline(torch, w)
        except Exception as e:  # keep the bench line even if the probe fails
            line["roofline"] = {"error": repr(e)}
        if not args.no_extras:
            extras = {}
            for s in w.schemes:
                if s == scheme:
                    continue
                P.integrate(prob, s, (x0,), w.t_final, w.steps)
                rr = P.integrate(prob, s, (x0,), w.t_final, w.steps)
                done = rr.diverged_at if rr.diverged else w.steps
                extras[s] = {"value": w.points * done / rr.device_seconds, "unit": UNIT,
                             "ms_per_time_step": 1e3 * rr.device_seconds / max(done, 1),
                             "diverged": rr.diverged, "diverged_at": rr.diverged_at, "reason": rr.reason}
            line["per_stepper"] = extras
            if world == 1:
                sample = args.cpu_sample_steps
                s_cpu, n_cpu = oracle_run(w, scheme, sample)
                line["cpu_baseline"] = {"value": w.points * n_cpu / s_cpu, "unit": UNIT, "cores": cpu_cores(),
                                        "kind": "port",
                                        "sample": f"{n_cpu} of {w.steps} {scheme} time steps on {w.extents} "
                                                  f"(oracle/cgl_oracle.py = reference algorithm on numpy/OpenBLAS)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    from paper_2403_02816_b200 import workloads as W
    w = W.CONFIGS[args.workload]
    scheme = args.scheme or w.schemes[0]
    if args.impl == "reference":
        reference_arm(args, w, scheme)
    else:
        gpu_arm(args, w, scheme)


if __name__ == "__main__":
    main()
