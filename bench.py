"""Benchmark of the CGL hot path on B200 (driver contract: one JSON line).

Headline workload (one workload for every N): BASELINE.json
configs[3] = C3, the 3D periodic cubic CGL on a 512^3 Fourier grid,
complex128, seeded random-phase u0, Lawson-RK4 (`if4`), tau = 0.01, 100 time
steps -- the largest configuration BASELINE times on one GPU, and slab-sharded
(distributed 3D FFT, NCCL all-to-all) at N > 1.  BASELINE quotes its metric on
no single config; C0, C1, C2 and C4 are reported as driver-clocked extras in
the same line (`per_config`).

One bench "step" = one full `integrate()` run of the workload (100 time
steps).  Metric = grid-point-steps/s = N_points * time_steps / second over the
stepping loop (the reference's timing scope, integrators.py:258-281; prepare
excluded).
  value   device time (CUDA events) of the loop, state resident in HBM (the
          2 GiB state is larger than L2; L2 is also flushed between runs);
          max over ranks.
  e2e     the public API with HOST buffers: pinned host state in, numpy out
          (H2D + loop + D2H inside the timed region).
  roofline  the dominant kernel of the step, timed live with CUDA events on its
          stream, against the measured HBM copy bandwidth (MEASURED_PEAKS.json);
          algorithmic bytes per launch are DESIGN.md's per-point figure x points.
  cpu_baseline  the CPU oracle port (numpy/OpenBLAS + pocketfft on all host
          threads; the reference algorithm, pinned to its outputs) on a bounded
          sample: time steps of the same workload, rank 0, N = 1.

--impl reference: the reference's CPU implementation of the path (the oracle
port; the reference is pure Python + numpy, /root/reference does not travel to
the box) on the same workload, rank 0 only.  That arm never imports the product
library.

--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (one process per GPU, NCCL).
"""

import argparse
import dataclasses
import json
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "grid-point-steps/s"
UNIT = "gp-steps/s"
# algorithmic HBM bytes per grid point per time step:
# Fourier if4 = 8 FFTs x 32 B + 7 extra 16-B operand reads; strang = 4 x 32 B
FOURIER_BYTES = {"if4": 368, "strang": 128}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--no-extras", action="store_true", help="skip per_config side runs and the CPU sample")
    ap.add_argument("--cpu-sample-steps", type=int, default=1,
                    help="time steps of the workload per CPU bench step (scaled up for small grids)")
    ap.add_argument("--time-steps", type=int, default=0, help="override the workload's step count")
    ap.add_argument("--sharded", action="store_true", help="use the slab-sharded 3D path even at N = 1")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def spawn_ranks(args):
    """`--gpus N` under plain python: re-exec under torch.distributed.run (one
    rank per GPU, rendezvous on 127.0.0.1); rank 0 prints the line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def workload(args):
    from paper_2403_02816_b200 import workloads as W  # host-side only: maps no library
    w = W.CONFIGS[args.workload]
    if args.time_steps:
        w = dataclasses.replace(w, steps=args.time_steps)
    return w, args.scheme or w.schemes[0]


def config_dict(w, scheme, world, parallelism=None):
    return {"workload": w.name, "grid": list(w.extents), "boundary": w.boundary, "scheme": scheme,
            "tau": w.tau, "time_steps": w.steps, "dtype": "complex128",
            "bench_step": f"one integrate() run = {w.steps} {scheme} time steps",
            "l2": "inputs larger than L2 (16 B x points per field); L2 also flushed (256 MiB write) between runs",
            "parallelism": parallelism or (f"replicas x{world}" if world > 1 else "single")}


# ---------------------------------------------------------------------------
# CPU side (oracle port): the reference arm and the cpu_baseline leg
# ---------------------------------------------------------------------------

def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample_steps(w, per_bench_step):
    """Time steps per CPU sample: `per_bench_step` at 512^3-class grids, more
    for small grids (about the same CPU work)."""
    return max(1, min(w.steps, int(per_bench_step * (1 << 27) / w.points)))


def oracle_run(w, scheme, max_steps):
    """The oracle port of the reference `integrate` on the workload's seeded
    input for at most `max_steps` steps; returns (loop seconds, steps done)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cgl_oracle as O
    from paper_2403_02816_b200 import workloads as W
    from threadpoolctl import threadpool_limits
    O.FFT_WORKERS = cpu_cores()
    p = O.Params(**{k: getattr(w.params, k) for k in O.Params.NAMES})
    u0 = W.initial_state(w)
    if w.boundary == "periodic":
        blocks = [O.FourierOp(O.symbol(w.extents, (w.interval,) * len(w.extents), p))]
        x0 = O._fftn(u0)
    else:
        a, b = w.interval
        d = len(w.extents)
        blocks = [O.KronOp([p.diffusion * O.FD_BUILDERS[w.boundary](n, b - a) + (p.alpha2 / d) * np.eye(n)
                            for n in w.extents])]
        x0 = u0
    del u0
    with threadpool_limits(limits=cpu_cores()):
        res = O.integrate(O.Prob(blocks, w.kind, p), scheme, (x0,), w.t_final, w.steps, max_steps=max_steps)
    done = res.diverged_at if res.diverged else min(w.steps, max_steps)
    return res.seconds, done


def cpu_sample_desc(w, scheme, n, cores):
    return (f"{n} of {w.steps} {scheme} time steps per sample on {list(w.extents)} (oracle/cgl_oracle.py: the "
            f"reference algorithm on numpy {np.__version__} + OpenBLAS zgemm, pocketfft via scipy.fft, "
            f"{cores} host threads)")


def reference_arm(args, w, scheme):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sample = cpu_sample_steps(w, args.cpu_sample_steps)
    # numpy has nothing to warm beyond the first call: one warm-up sample at most
    # (a 512^3 time step is tens of seconds of CPU work)
    for _ in range(min(args.warmup, 1)):
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
        "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * tot_s / args.steps,
        "ms_per_time_step": 1e3 * tot_s / max(tot_steps, 1),
        "higher_is_better": True, "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic", "config": config_dict(w, scheme, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": cpu_sample_desc(w, scheme, sample, cores)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def hbm_peak():
    """(GB/s, source): the measured copy bandwidth, else the recipe's fallback."""
    pk = peaks()
    for k in ("hbm_gbs", "hbm_gbps", "hbm_copy_gbps"):
        if k in pk:
            return float(pk[k]), f"MEASURED_PEAKS.json {k}"
    return 6540.5, "fallback (SURVEY.md 0.5 measured copy bandwidth)"


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


def fourier_roofline(torch, w, scheme, step_seconds):
    """Pencil-FFT passes of the Fourier step (csrc/fftpass.cu), each timed live
    per launch with CUDA events (10 launches inside a captured graph, fields
    refilled from a pristine copy whose own time is subtracted, so g and the
    flows see realistic values) on the workload's 512^3 grid.  `achieved` is
    the DOMINANT kernel's (largest share of the step: the fused g pass of if4,
    the end-of-step flow pass of strang) algorithmic HBM bytes per launch --
    32 B/pt for a transform pass, + 16 B per extra operand read or written
     -- over its launch time; every pass rides along in `passes`,
    and the whole-step rate on the 368 / 128 B/pt algorithmic traffic of
    SURVEY.md 8(d) in `step_level`."""
    from paper_2403_02816_b200 import SCHEMES, workloads as W
    from paper_2403_02816_b200.plan import PencilFourierPlan
    peak, src = hbm_peak()
    n = w.points
    prob = W.build_problem(w)
    prob.prepare(w.tau, SCHEMES[scheme])
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.empty(w.extents, dtype=torch.complex128, device="cuda")
    x.real.normal_(generator=g)
    x.imag.normal_(generator=g)
    plan = PencilFourierPlan(prob, scheme, [x])
    plan.load_state([x], w.tau)
    plan.flag = None          # timing only: no divergence bookkeeping
    from paper_2403_02816_b200 import fftpass
    T0 = fftpass.fftn(0.1 * x)  # coefficients of an O(0.1) field, as in C3
    T = T0.clone()
    u = x.clone()
    gs = [x.clone()]   # the accumulated Lawson combination
    reps = 10
    copy_dt = _time(torch, _graphed(torch, lambda: [T.copy_(T0) for _ in range(reps)]), reps=3) / reps

    def per_launch(fn):
        return _time(torch, _graphed(torch, lambda: [(T.copy_(T0), fn()) for _ in range(reps)]), reps=3) / reps - copy_dt
    last = len(w.extents) - 1
    if scheme == "if4":
        progs = {"g (axis 0: F^-1, g, F)": (lambda: plan._pass("g", 0, T, T, w.tau, scale=1.0 / n), 32, 4),
                 "plain axis 1": (lambda: plan._pass("plain", 1, T, T, w.tau), 32, 8),
                 "if4_b1 (axis 2)": (lambda: plan._pass("if4_b1", last, T, T, w.tau, u=u, g_out=gs[0]), 64, 1),
                 "if4_b3 (axis 2)": (lambda: plan._pass("if4_b3", last, T, T, w.tau, u=u, g=(gs[0], None, None),
                                                        g_out=gs[0]), 80, 2),
                 "if4_b4 (axis 2)": (lambda: plan._pass("if4_b4", last, T, T, w.tau, u=gs[0], u_out=u), 64, 1)}
        dom = "g (axis 0: F^-1, g, F)"
    else:
        y = x.clone()
        a0 = "str_a0f" if plan._fused_boundary() else "str_a0"
        progs = {"str_a0 (axis 0: F^-1, 2 flows, check, F)": (
                     lambda: plan._pass(a0, 0, T, T, w.tau, u_out=y, scale=1.0 / n), 48, 1),
                 "plain axis 1": (lambda: plan._pass("plain", 1, T, T, w.tau), 32, 2),
                 "str_mid (axis 2: F, E1, F^-1)": (lambda: plan._pass("str_mid", last, T, T, w.tau), 32, 1)}
        dom = "str_a0 (axis 0: F^-1, 2 flows, check, F)"
    passes = {}
    for name, (fn, bpp, per_step) in progs.items():
        dt = per_launch(fn)
        a = bpp * n / dt / 1e9
        passes[name] = {"ms": dt * 1e3, "bytes_per_point": bpp, "launches_per_step": per_step, "gbs": a,
                        "frac": a / peak}
    d = passes[dom]
    step_bytes = FOURIER_BYTES.get(scheme, 0) * n
    # DRAM bytes per launch of the dominant program from the ncu --set full capture of this
    # round at 512^3 (if4: fft_r32_kernel, profiles/r02e_fft_r32.txt; strang: profiles/r02c_fft_passes.txt;
    # dram__bytes_read.sum + dram__bytes_write.sum)
    traffic = {"if4": 2.147565e9 + 2.119455e9, "strang": 2.149681e9 + 4.291060e9}.get(scheme) \
        if tuple(w.extents) == (512, 512, 512) else None
    return {"bound": "hbm", "achieved": d["gbs"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
            "traffic": traffic,
            "kernel": f"cgl::fftp::fft_*_kernel, dominant program: {dom} (largest share of the step in "
                      "profiles/r02f_launches_C3_if4.txt / _strang.txt: the largest single kernel instantiation; the 8 plain axis-1 passes together are 34 % at 0.80 of the peak)",
            "algorithmic_bytes_per_launch": d["bytes_per_point"] * n, "per_launch_ms": d["ms"], "peak_source": src,
            "passes": passes,
            "step_level": {"algorithmic_bytes_per_step": step_bytes,
                           "achieved_gbps": step_bytes / step_seconds / 1e9 if step_seconds else None,
                           "frac": step_bytes / step_seconds / 1e9 / peak if step_seconds else None}}


def step_roofline(w, scheme, step_seconds):
    peak, src = hbm_peak()
    step_bytes = FOURIER_BYTES.get(scheme, 0) * w.points
    a = step_bytes / step_seconds / 1e9
    return {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak, "traffic": None,
            "kernel": f"whole {scheme} time step (algorithmic {FOURIER_BYTES.get(scheme)} B/pt)",
            "peak_source": src}


def gemm_roofline(torch, w, scheme_fields=2):
    """C1's dominant kernel: the 2-field axis-0 product E1/2 [u, g1] of the
    quad-form if4 step on the INT8 tensor cores (ozgemm_persistent_kernel),
    timed per launch inside a captured graph, data pre-sliced as in the step.
    Executed int8 MACs (block skipping counted out) against the dense INT8
    tcgen05 rate measured on this pool (tools/mma_rate.cu: 8192 MAC/clk/SM)
    at the sampled SM clock, plus 2 x bf16 from MEASURED_PEAKS.json."""
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
    ozaki.mode_product_oz(ins, [fac] * scheme_fields, outs, 0, ws)
    Q = w.points // n
    per = lib.cgl_oz_slice_bytes(ozaki.S, Q, n, 0)
    Bs = [ws.bufs[("D", f, n)][0] for f in range(scheme_fields)]
    Be = [ws.bufs[("D", f, n)][1] for f in range(scheme_fields)]

    def gemm_only():
        _lib.check(lib.cgl_oz_gemm(_lib.stream(), ozaki.S, n, Q, n, scheme_fields,
                                   _lib.ptr_array([fac.A] * scheme_fields), _lib.ptr_array([fac.Ae] * scheme_fields),
                                   _lib.ptr_array([fac.Az] * scheme_fields), _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                   None, _lib.ptr_array(outs), Q, 1, 0, 0, per, Q, n * Q, None, 0), "oz_gemm")
    reps_in_graph = 10

    def gemm_rep():
        for _ in range(reps_in_graph):
            gemm_only()
    dt = _time(torch, _graphed(torch, gemm_rep)) / reps_in_graph
    bn = ozaki.geometry()[1]
    macs = ozaki.executed_macs_left(fac, (Q + bn - 1) // bn, scheme_fields)
    props = torch.cuda.get_device_properties(0)
    sm_mhz = 1965.0
    mma_peak = 2.0 * 8192 * props.multi_processor_count * sm_mhz * 1e6 / 1e12
    achieved = 2.0 * macs / dt / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": mma_peak, "unit": "TOPS (int8)",
            "frac": achieved / mma_peak, "per_launch_ms": dt * 1e3,
            "kernel": "ozgemm_persistent_kernel<8,32,4>: 2-field axis-0 product of the C1 if4 step",
            "peak_source": "tools/mma_rate.cu measured tcgen05 kind::i8 rate 8192 MAC/clk/SM x 148 SMs x 1965 MHz",
            "frac_vs_2x_bf16": achieved / (2.0 * peaks().get("bf16_tflops", 1640.0))}


def launches(lib, prob):
    return lib.cgl_launch_count() + sum(fp.replayed_launches for fp in getattr(prob, "_plans", {}).values())


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
    x0 = W.state_for_problem(w, W.initial_state_device(w))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(args.warmup):
        r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    l0 = launches(lib, prob)
    dev_total = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
            dev_total += r.device_seconds
    n_launch = launches(lib, prob) - l0
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([dev_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_total = float(t.item())
    steps_done = (r.diverged_at if r.diverged else w.steps)
    value = world * w.points * steps_done * args.steps / dev_total

    # e2e through the public API with host buffers (pinned host tensor in, numpy out)
    x_pinned = x0.cpu().pin_memory()
    P.integrate(prob, scheme, (x_pinned,), w.t_final, w.steps)
    e2e_total = 0.0
    r2 = None
    for _ in range(args.steps):
        r2 = None  # the previous result's page-locked block goes back to torch's host cache
        flush.zero_()
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
    del x_pinned, r2

    step_s = dev_total / args.steps / max(steps_done, 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_total / args.steps,
        "ms_per_time_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(w, scheme, world),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16 * w.points,
                "d2h_bytes_per_step": 16 * w.points, "ms_per_step": 1e3 * e2e_total / args.steps},
        "gpu_launches": int(n_launch),
        "clocks": clk.summary(),
        "diverged": bool(r.diverged),
    }
    if rank == 0:
        try:
            if w.boundary == "periodic":
                line["roofline"] = fourier_roofline(torch, w, scheme, step_s)
            else:
                line["roofline"] = gemm_roofline(torch, w)
        except Exception as e:  # keep the bench line even if the probe fails
            line["roofline"] = {"error": repr(e)}
            if w.boundary == "periodic":
                line["roofline"].update(step_roofline(w, scheme, step_s))
        del prob, x0, r
        if not args.no_extras and world == 1:
            line["per_config"] = per_config(torch, P, W, skip=(w.name, scheme))
            sample = cpu_sample_steps(w, args.cpu_sample_steps)
            s_cpu, n_cpu = oracle_run(w, scheme, sample)
            line["cpu_baseline"] = {"value": w.points * n_cpu / s_cpu, "unit": UNIT, "cores": cpu_cores(),
                                    "kind": "port", "sample": cpu_sample_desc(w, scheme, n_cpu, cpu_cores())}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


EXTRAS = (("C0", "strang", None), ("C1", "if4", None), ("C1", "strang", None), ("C1", "rk4", None),
          ("C1", "rk4", 0.001), ("C2", "split4", None), ("C3", "strang", None), ("C4", "if4", None))


def per_config(torch, P, W, skip=()):
    """Every other BASELINE config, one warm run + one timed run each
    (device time of the full integrate() loop)."""
    out = {}
    for cfg, scheme, tau in EXTRAS:
        w = W.CONFIGS[cfg]
        if (w.name, scheme) == skip and tau is None:
            continue
        if tau is not None:
            w = dataclasses.replace(w, tau=tau)
        key = f"{cfg}/{scheme}" + (f"@tau={tau}" if tau else "")
        try:
            prob = W.build_problem(w)
            x0 = W.state_for_problem(w, W.initial_state_device(w))
            P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
            r = P.integrate(prob, scheme, (x0,), w.t_final, w.steps)
            done = r.diverged_at if r.diverged else w.steps
            out[key] = {"value": w.points * done / r.device_seconds, "unit": UNIT,
                        "ms_per_time_step": 1e3 * r.device_seconds / max(done, 1), "time_steps": w.steps,
                        "grid": list(w.extents), "tau": w.tau, "diverged": bool(r.diverged),
                        "diverged_at": int(r.diverged_at), "reason": r.reason}
            del prob, x0, r
        except Exception as e:
            out[key] = {"error": repr(e)}
        torch.cuda.empty_cache()
    return out


def sharded_arm(args, w, scheme):
    """3D configs at N > 1: axis-0 slab sharding (FD: all-to-all transposes
    around the axis-0 product; Fourier: distributed 3D FFT).  Strong scaling:
    the global grid is fixed; value = global points x steps / max-over-ranks
    device time of the stepping loop."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    else:
        group = None
    from paper_2403_02816_b200 import SCHEMES, _lib, distributed as D, slabfourier as SF, workloads as W
    from paper_2403_02816_b200.spectral import dft_forward, dft_inverse
    lib = _lib.load()
    prob = W.build_problem(w)
    u0 = W.initial_state_device(w)
    steps = w.steps
    if w.boundary == "periodic":
        prob.prepare(w.tau, SCHEMES[scheme])
        uhat = dft_forward(u0)
        layout = "cols" if scheme == "if4" else "slabs"
        x_local = SF.split_global(uhat if scheme == "if4" else dft_inverse(uhat), world, layout)[rank]
        del uhat
        plan = SF.ShardedFourierPlan(prob, scheme, w.extents, world, [rank], group)

        def run(x):
            e0, e1 = _events(torch)
            e0.record()
            key = plan.run([x], steps, w.tau)
            e1.record()
            torch.cuda.synchronize()
            out = plan.U[0] if scheme == "if4" else plan.Us[steps % 2][0]
            return e0.elapsed_time(e1) / 1e3, key, out
    else:
        L = D.SlabLayout(w.extents, world)
        a, b = L.bounds(rank)
        x_local = u0[a:b].contiguous()

        def run(x):
            out, _, _, dt = D.integrate_sharded(prob, scheme, [x], w.t_final, steps, L, group)
            return dt, None, out[0]
    del u0
    torch.cuda.empty_cache()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        run(x_local)
    l0 = lib.cgl_launch_count()
    total = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if group is not None:
                dist.barrier()
            dt, _, _ = run(x_local)
            total += dt
    n_launch = lib.cgl_launch_count() - l0
    # e2e: this rank's share of the state from pinned host memory, result back to host
    x_host = x_local.cpu().pin_memory()
    e2e_total = 0.0
    for _ in range(args.steps):
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0 = time.perf_counter()
        xd = x_host.to("cuda", non_blocking=True)
        _, _, out = run(xd)
        _ = out.cpu().numpy()
        torch.cuda.synchronize()
        e2e_total += time.perf_counter() - t0
    t = torch.tensor([total, e2e_total], dtype=torch.float64, device="cuda")
    if group is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total, e2e_total = float(t[0]), float(t[1])
    value = w.points * steps * args.steps / total
    if rank == 0:
        step_s = total / args.steps / steps
        cfg = config_dict(w, scheme, world, parallelism=f"axis-0 slabs x{world}")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "ms_per_time_step": 1e3 * step_s,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
                "data": "synthetic", "config": cfg,
                "e2e": {"value": w.points * steps * args.steps / e2e_total, "unit": UNIT,
                        "h2d_bytes_per_step": 16 * x_local.numel(), "d2h_bytes_per_step": 16 * x_local.numel(),
                        "per": "rank (every rank copies its slab)"},
                "gpu_launches": int(n_launch), "clocks": clk.summary()}
        if w.boundary == "periodic":
            rl = step_roofline(w, scheme, step_s * world)
            rl["note"] = "per-rank HBM rate: algorithmic bytes of the rank's 1/N share over the step time"
            line["roofline"] = rl
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    _, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    w, scheme = workload(args)
    if args.impl == "reference":
        reference_arm(args, w, scheme)
    elif (world > 1 or args.sharded) and len(w.extents) == 3:
        sharded_arm(args, w, scheme)
    else:
        gpu_arm(args, w, scheme)


if __name__ == "__main__":
    main()
