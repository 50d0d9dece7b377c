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
    ap.add_argument("--time-steps", type=int, default=0, help="override the workload's step count (3D configs)")
    ap.add_argument("--sharded", action="store_true", help="use the slab-sharded 3D path even at N = 1")
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
    sample = max(1, int((args.cpu_sample_steps // 3) * (1 << 18) / w.points))
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


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time(torch, fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = _events(torch)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def _graphed(torch, fn):
    """fn captured once into a CUDA graph; returns the replay callable."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    return g.replay


def gemm_roofline(torch, w, scheme_fields=2):
    """Dominant kernel of the if4 step: the 2-field axis-0 (left-form) product
    of the quad-form step ([A, G] = E1/2 [u, g1]; all four products of a step
    are 2-field)
    on the INT8 tensor cores (ozgemm_persistent_kernel), timed per launch with CUDA
    events on the workload shapes, data pre-sliced as in the step.  Reported
    against the INT8 dense tensor peak on EXECUTED int8 MACs (block skipping
    counted out), plus the FP64-equivalent view against the measured DMMA
    peak (what the FP64 tensor path could reach on the same product)."""
    from paper_2403_02816_b200 import _lib, ozaki, workloads as W
    lib = _lib.load()
    n = w.extents[0]
    prob = W.build_problem(w)
    prob.operator.prepare(w.tau, (1,))
    fac = prob.operator.sliced_factors(1)[0]
    g = torch.Generator(device="cuda").manual_seed(0)
    ins = [torch.randn(w.extents, dtype=torch.complex128, device="cuda", generator=g) for _ in range(scheme_fields)]
    outs = [torch.empty_like(x) for x in ins]
    ws = ozaki.Workspace()
    ozaki.mode_product_oz(ins, [fac] * scheme_fields, outs, 0, ws)  # slices the data into ws
    Q = w.points // n
    per = lib.cgl_oz_slice_bytes(ozaki.S, Q, n, 0)
    Bs = [ws.bufs[("D", f, n)][0] for f in range(scheme_fields)]
    Be = [ws.bufs[("D", f, n)][1] for f in range(scheme_fields)]

    def gemm_only():
        _lib.check(lib.cgl_oz_gemm(_lib.stream(), ozaki.S, n, Q, n, scheme_fields,
                                   _lib.ptr_array([fac.A] * scheme_fields), _lib.ptr_array([fac.Ae] * scheme_fields),
                                   _lib.ptr_array([fac.Az] * scheme_fields), _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                   None, _lib.ptr_array(outs), Q, 1, 0, 0, per, Q, n * Q, None, 0), "oz_gemm")
    # per-launch time as in the step: 10 back-to-back launches inside one
    # captured graph (programmatic dependent launch between them, no
    # graph-launch gap), event time / 10
    reps_in_graph = 10

    def gemm_rep():
        for _ in range(reps_in_graph):
            gemm_only()

    def product_rep():
        for _ in range(reps_in_graph):
            ozaki.mode_product_oz(ins, [fac] * scheme_fields, outs, 0, ws)
    dt = _time(torch, _graphed(torch, gemm_rep)) / reps_in_graph
    dt_with_slicing = _time(torch, _graphed(torch, product_rep)) / reps_in_graph
    bn = ozaki.geometry()[1]
    macs = ozaki.executed_macs_left(fac, (Q + bn - 1) // bn, scheme_fields)
    dense = ozaki.dense_macs(n, Q, n, scheme_fields)
    # live FP64 DMMA peak
    stream = _lib.stream()
    lib.cgl_probe_dmma(stream, 256)
    best = 0.0
    for _ in range(3):
        e0, e1 = _events(torch)
        e0.record()
        fl = lib.cgl_probe_dmma(stream, 4096)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, fl / (e0.elapsed_time(e1) / 1e3) / 1e12)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    int8_peak = 2.0 * peaks["bf16_tflops"]
    achieved = 2.0 * macs / dt / 1e12
    fp64_alg = 8.0 * n * w.points * scheme_fields / dt / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TOPS (int8)",
            "frac": achieved / int8_peak,
            # dram__bytes_read.sum + dram__bytes_write.sum of one 2-field launch, ncu --set full
            # (profiles/r01f_ncu_full_step_kernels.txt; ncu flushes caches, so this is the
            # cold upper bound -- in the step the operands are L2-resident)
            "traffic": 9.947392e6, "traffic_unit": "bytes per launch",
            "traffic_source": "profiles/r01g_ncu_full_step_kernels.txt (cold-cache ncu capture)",
            "kernel": "ozgemm_persistent_kernel<8,32,4> (tcgen05.mma kind::i8, double-buffered TMEM level "
                      "accumulators): 2-field axis-0 product of the if4 step (E1/2 [u, g1]), M=N=K=512 complex "
                      "per field, "
                      "S=8 int8 slices",
            "per_launch_ms": dt * 1e3, "per_launch_ms_incl_data_slicing": dt_with_slicing * 1e3,
            "executed_int8_macs_per_launch": macs, "dense_int8_macs_per_launch": dense,
            "block_skip_fraction": 1.0 - macs / dense,
            "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (dense INT8 = 2x BF16 on B200, "
                           "B200_PROFILING.md nominal table); no measured INT8 figure exists",
            "fp64_equivalent": {"achieved_tflops": fp64_alg, "dmma_peak_tflops": best,
                                "ratio_vs_dmma_peak": fp64_alg / best,
                                "note": "algorithmic 8*n flops per point per product; the FP64 tensor path "
                                        "(zgemm_kernel, DMMA) reaches ~32 TFLOP/s on this product"}}


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
                # bounded CPU sample: ~24 C1-sized time steps worth of work
                sample = max(1, int(args.cpu_sample_steps * (1 << 18) / w.points))
                s_cpu, n_cpu = oracle_run(w, scheme, sample)
                line["cpu_baseline"] = {"value": w.points * n_cpu / s_cpu, "unit": UNIT, "cores": cpu_cores(),
                                        "kind": "port",
                                        "sample": f"{n_cpu} of {w.steps} {scheme} time steps on {w.extents} "
                                                  f"(oracle/cgl_oracle.py = reference algorithm on numpy/OpenBLAS)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def sharded_arm(args, w, scheme):
    """3D configs at N > 1: axis-0 slab sharding (FD: NCCL all-to-all inside the
    axis-0 mode product; Fourier: distributed 3D FFT).  Strong scaling: the
    global grid is fixed; value = global points x steps / max-over-ranks time."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_02816_b200 import SCHEMES, distributed as D, slabfourier as SF, workloads as W
    from paper_2403_02816_b200.spectral import dft_forward, dft_inverse
    steps = args.time_steps or w.steps
    wl = w.scaled(w.extents[0], steps) if steps != w.steps else w
    prob = W.build_problem(wl)
    u0 = W.initial_state_device(wl)
    times = []
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        if wl.boundary == "periodic":
            prob.prepare(wl.tau, SCHEMES[scheme])
            uhat = dft_forward(u0)
            plan = SF.ShardedFourierPlan(prob, scheme, wl.extents, world, [rank], dist.group.WORLD)
            x0 = SF.split_global(uhat if scheme == "if4" else dft_inverse(uhat), world,
                                 "cols" if scheme == "if4" else "slabs")[rank:rank + 1]
            del uhat
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.run(x0, steps, wl.tau)
            e1.record()
            torch.cuda.synchronize()
            dt = e0.elapsed_time(e1) / 1e3
        else:
            L = D.SlabLayout(wl.extents, world)
            a, b = L.bounds(rank)
            x0 = [u0[a:b].contiguous()]
            _, _, _, dt = D.integrate_sharded(prob, scheme, x0, wl.t_final, steps, L, dist.group.WORLD)
        if it >= args.warmup:
            times.append(dt)
    t = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t.item())
    value = wl.points * steps * args.steps / total
    if rank == 0:
        cfg = config_dict(wl, scheme, world)
        cfg["parallelism"] = f"axis-0 slabs x{world}"
        print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
                          "config": cfg}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    from paper_2403_02816_b200 import workloads as W
    w = W.CONFIGS[args.workload]
    scheme = args.scheme or w.schemes[0]
    _, world, _ = dist_env()
    if args.impl == "reference":
        reference_arm(args, w, scheme)
    elif (world > 1 or args.sharded) and len(w.extents) == 3:
        sharded_arm(args, w, scheme)
    else:
        gpu_arm(args, w, scheme)


if __name__ == "__main__":
    main()
