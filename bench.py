"""bench.py -- headline benchmark of the JACC B200 hot path.

Workload (BASELINE.json configs[1]): Jacobi-2D fp64 16384 x 16384, 100
timesteps = 200 `parallel loop` launches per step, owned row blocks over N
devices with HALO (boundary-row dirty-range) merge.  Metric: algorithmic
loop GB/s (8 B read per src element + 8 B written per interior dst element
per launch), whole job.  Inputs (2 x 2 GiB) are far larger than L2, so no
explicit flush is needed between timed iterations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl jacc|reference]

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (the
only reference this tier has) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GRID = 16384
TSTEPS = 100
METRIC = "loop GB/s (Jacobi-2D fp64 16384^2, 100 timesteps, HALO merge)"
UNIT = "GB/s"


def algo_bytes_per_sweep(N, n):
    """Algorithmic HBM bytes of one Jacobi launch summed over devices: each
    device reads its owned rows plus one halo row each side (8 B/element)
    and writes its interior elements (8 B/element)."""
    tot = 0
    for d in range(n):
        q, r = divmod(N, n)
        lo = d * q + min(d, r)
        hi = (d + 1) * q + min(d + 1, r)
        i0, i1 = max(lo, 1), min(hi, N - 1)
        if i1 <= i0:
            continue
        tot += 8 * N * (i1 - i0 + 2) + 8 * (i1 - i0) * (N - 2)
    return tot


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


HBM_SPEC_GBS = 8000.0      # B200 datasheet HBM3e
FP64_SPEC_TFLOPS = 40.0    # B200 datasheet fp64 (tensor), SURVEY 8(d)


def load_dgemm_peak():
    """cuBLAS DGEMM 8192^3 measured on this pool (tools/probe_box.py ->
    profiles/probe_box_r*.json): the fp64 tensor-pipe reference."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "probe_box_r*.json")), reverse=True):
        with open(p) as f:
            j = json.load(f)
        if j.get("dgemm_tflops"):
            return float(j["dgemm_tflops"]), os.path.basename(p)
    return None, None


def load_traffic(kernel="jacobi2d"):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")), reverse=True):
        try:
            with open(p) as f:
                j = json.load(f)
            k = j.get("kernels", {}).get(kernel)
            if k and k.get("dram_bytes_per_launch"):
                return float(k["dram_bytes_per_launch"]), os.path.basename(p)
        except Exception:
            pass
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, cuda_ords):
        # nvidia-smi indices of every GPU the job uses (through
        # CUDA_VISIBLE_DEVICES when it remaps ordinals)
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        vis = [v.strip() for v in vis.split(",")] if vis else []
        idx = [vis[o] if o < len(vis) and vis[o].isdigit() else str(o) for o in cuda_ords]
        self.idx = ",".join(idx)
        self.samples = []
        self.proc = None
        self.window = None

    def mark(self, t0, t1):
        """restrict the summary to samples taken in [t0, t1] (time.monotonic);
        the sampler is started before the warm-up so nvidia-smi's own start-up
        (seconds with several ranks on the box) never leaves it unsampled"""
        self.window = (t0, t1)

    def __enter__(self):
        if not self.idx:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.monotonic(), parts))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        samples = [p for _, p in self.samples]
        where = "timed region"
        if self.window:
            t0, t1 = self.window
            inside = [p for t, p in self.samples if t0 <= t <= t1]
            if not inside:  # region shorter than the 100 ms period: nearest samples
                inside = [p for t, p in self.samples if t0 - 0.25 <= t <= t1 + 0.25]
                where = "timed region +-250 ms"
            samples = inside
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for s in samples:
            try:
                util = float(s[6])
                if util > 50:
                    sm.append(float(s[0]))
                mx = float(s[1])
            except ValueError:
                continue
            for k, name in enumerate(names):
                if s[2 + k].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(samples), "window": where}


# ----------------------------------------------------------------------------
# reference arm / cpu baseline: the CPU oracle on a bounded sample
# ----------------------------------------------------------------------------
_ORC_GRID = None


def oracle_sample(sweeps):
    """Time `sweeps` oracle launches of the J16K sweep on the full 16384^2
    grid (single thread).  Returns (GB/s algorithmic, seconds, sample text)."""
    global _ORC_GRID
    import __graft_entry__ as ge
    ge.build_oracle()
    ge.build_synth()
    import oracle as orc
    import synth
    if _ORC_GRID is None:
        _ORC_GRID = synth.polybench_jacobi2d(N_GRID)
    A, B = _ORC_GRID
    t0 = time.perf_counter()
    src, dst = A, B
    for _ in range(sweeps):
        orc.jacobi2d_sweep(src, dst)
        src, dst = dst, src
    dt = time.perf_counter() - t0
    gbs = sweeps * algo_bytes_per_sweep(N_GRID, 1) / dt / 1e9
    return gbs, dt, f"{sweeps} oracle sweeps of the 16384^2 grid (of 200 per step), 1 thread"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sweeps = 2
    for _ in range(args.warmup):
        oracle_sample(1)
    vals, times = [], []
    for _ in range(args.steps):
        g, dt, sample = oracle_sample(sweeps)
        vals.append(g)
        times.append(dt)
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3 * (2 * TSTEPS / sweeps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (PolyBench jacobi-2d init)",
        "config": {"workload": "J16K: Jacobi-2D fp64 16384x16384, 100 timesteps",
                   "sample": sample, "l2": "inputs 2x2 GiB >> 126 MB L2"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# the CUDA path
# ----------------------------------------------------------------------------
class Ctx:
    """Launch context: single process (N logical devices, real or virtual
    GPUs) or one process per GPU under torch.distributed.run (C-ABI
    multi-process mode: CUDA-IPC peer replicas, NCCL for reductions)."""

    def __init__(self, J, torch, n):
        self.J, self.torch, self.n = J, torch, n
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.mp = self.world > 1
        ngpu = torch.cuda.device_count()
        if self.mp:
            import torch.distributed as dist
            from paper_2110_14340_b200 import dist as jd
            self.dist, self.jd = dist, jd
            if self.world != n:
                raise SystemExit(f"--gpus {n} must equal WORLD_SIZE {self.world}")
            dist.init_process_group("gloo", init_method="env://")
            lr = int(os.environ.get("LOCAL_RANK", str(self.rank)))
            ordv = lr % ngpu
            torch.cuda.set_device(ordv)
            _, _, distinct = jd.init_rank(ordv)
            self.virtual = not distinct
            self.local = [self.rank]
            self.ords = [ordv]
            self.all_ords = sorted({r % ngpu for r in range(self.world)})
        else:
            self.virtual = ngpu < n
            self.ords = list(range(n)) if not self.virtual else [0] * n
            J.jacc_init(n, self.ords)
            self.local = list(range(n))
            self.all_ords = sorted(set(self.ords))
        self.streams = {}
        for d in self.local:
            sp, o = J.jacc_get_stream(d)
            self.streams[d] = (torch.cuda.ExternalStream(sp, device=f"cuda:{o}"), o)

    def create(self, arr):
        if self.mp:
            self.jd.data_create(arr)
        else:
            self.J.jacc_data_create(arr)

    def sync(self):
        for o in sorted(set(o for _, o in self.streams.values())):
            self.torch.cuda.synchronize(o)

    def barrier(self):
        if self.mp:
            self.dist.barrier()

    def reduce(self, x, op="max"):
        if not self.mp:
            return x
        t = self.torch.tensor([float(x)], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def timed(self, fn, reps):
        """Device time of reps x fn (CUDA events on every local stream, max
        over local devices, then max over ranks)."""
        torch = self.torch
        self.J.jacc_wait()
        self.sync()
        self.barrier()
        st, en = {}, {}
        for d, (s, o) in self.streams.items():
            with torch.cuda.device(o):
                st[d] = torch.cuda.Event(enable_timing=True)
                en[d] = torch.cuda.Event(enable_timing=True)
                st[d].record(s)
        for _ in range(reps):
            fn()
        for d, (s, o) in self.streams.items():
            with torch.cuda.device(o):
                en[d].record(s)
        self.J.jacc_wait()
        self.sync()
        t = max(st[d].elapsed_time(en[d]) for d in self.streams) / 1e3
        return self.reduce(t, "max")

    def finalize(self):
        if self.mp:
            self.jd.finalize()
            self.dist.destroy_process_group()
        else:
            self.J.jacc_finalize()


def run_jacc(args):
    import torch
    import __graft_entry__ as ge
    ge.build_synth()
    ge.build_jacc()
    import synth
    from paper_2110_14340_b200 import jacc as J

    n = args.gpus
    C = Ctx(J, torch, n)
    N = N_GRID
    A, B = synth.polybench_jacobi2d(N)
    J.jacc_set_merge_policy(J.JACC_MERGE_HALO if args.merge == "halo" else J.JACC_MERGE_EAGER)
    for arr in (A, B):
        C.create(arr)
        J.jacc_update_device(arr)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    args_ab = [J.arg(IN, A), J.arg(OUT, B)]
    args_ba = [J.arg(IN, B), J.arg(OUT, A)]

    def step():
        for _ in range(TSTEPS):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, args_ab, 0)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, args_ba, 0)

    clk = ClockSampler(C.all_ords if C.rank == 0 else []).__enter__()  # rank 0 samples all GPUs
    for _ in range(args.warmup):
        step()
    # host cost of issuing one launch (plan + enqueue on every device), timed
    # while the GPU is still busy with earlier work (asynchronous launches)
    C.sync()
    h0 = time.perf_counter()
    step()
    host_us = (time.perf_counter() - h0) / (2 * TSTEPS) * 1e6
    J.jacc_wait()
    # kernel-level timing (CUDA events around every launch on its stream)
    J.jacc_set_profiling(1)
    J.jacc_profile_reset()
    t_plain = C.timed(step, 1)
    kern = {d: J.jacc_profile_totals(d) for d in C.local}
    J.jacc_set_profiling(0)
    # the timed steps replay one CUDA graph of the 200-launch step (captured
    # at steady state: identical device work, host planning amortised);
    # multi-process mode has no graphs and issues the launches directly
    use_graph = not C.mp and not args.no_graph
    if use_graph:
        J.jacc_graph_begin()
        step()
        gid = J.jacc_graph_end()
        J.jacc_graph_replay(gid, 1)  # warm the graph
        timed_step = lambda: J.jacc_graph_replay(gid, 1)
    else:
        timed_step = step
    w0 = time.monotonic()
    t = C.timed(timed_step, args.steps)
    clk.mark(w0, time.monotonic())
    clk.__exit__()
    bytes_step = 2 * TSTEPS * algo_bytes_per_sweep(N, n)
    value = bytes_step * args.steps / t / 1e9
    # kernels per timed step: one loop kernel per device per launch (HALO
    # boundary pushes are fused into it), plus one merge kernel per device
    # per launch under EAGER with n > 1
    per_launch = 1 + (1 if (args.merge == "eager" and n > 1) else 0)
    launches = C.reduce(sum(k[2] for k in kern.values()), "sum") * per_launch * args.steps
    # dominant kernel: jacobi2d; average launch duration on the slowest device
    k_avg = C.reduce(max(k[0] / max(k[2], 1) for k in kern.values()), "max")
    per_dev_bytes = algo_bytes_per_sweep_dev(N, n, 0)
    achieved = per_dev_bytes / k_avg / 1e9
    peak, peak_src = load_peaks()
    traffic, tsrc = load_traffic("jacobi2d")
    if traffic is not None and n > 1:
        traffic = None  # the committed capture is of the n=1 launch

    # ---- e2e through the public API with host buffers ----
    e2e_times = []
    for it in range(max(1, min(args.steps, 3)) + 1):
        C.sync()
        C.barrier()
        t0 = time.perf_counter()
        J.jacc_update_device(A)
        J.jacc_update_device(B)
        step()
        J.jacc_update_host(A)
        t1 = time.perf_counter()
        if it > 0:
            e2e_times.append(C.reduce(t1 - t0, "max"))
    e2e = bytes_step / statistics.median(e2e_times) / 1e9

    extra = {}
    if args.extra and not C.mp:
        extra = run_extra_loops(J, C, n, peak)
    C.finalize()
    if args.extra and not C.mp and n == 1:
        extra["eager_merge_2virtual"] = eager_merge_probe(J, torch, A, B)

    cpu = None
    if args.cpu_baseline and n == 1 and C.rank == 0:
        g, dt, sample = oracle_sample(args.cpu_sweeps)
        cpu = {"value": g, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
               "seconds": dt}
    if C.rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (PolyBench jacobi-2d init, seeded generators in synth/)",
        "config": {"workload": "J16K: Jacobi-2D fp64 16384x16384, 100 timesteps (200 launches/step)",
                   "merge": args.merge, "launch": "one process per GPU" if C.mp else "single process",
                   "issue": "CUDA graph replay of the captured step" if use_graph else "jacc_launch x200",
                   "ms_per_step_plain_launches": t_plain * 1e3,
                   "host_us_per_launch": host_us,
                   "virtual_devices": C.virtual,
                   "l2": "no flush: inputs 2x2 GiB >> 126 MB L2",
                   "parallelism": f"row-block owner partition over {n} device(s)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "frac_of_spec": achieved / HBM_SPEC_GBS, "spec_peak": HBM_SPEC_GBS,
                     "kernel": "jacobi2d_kernel", "kernel_avg_us": k_avg * 1e6,
                     "algo_bytes_per_launch": per_dev_bytes, "peak_source": peak_src,
                     "traffic_source": tsrc},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 2 * A.nbytes,
                "d2h_bytes_per_step": A.nbytes},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if extra:
        line["loops"] = extra
    print(json.dumps(line), flush=True)


def algo_bytes_per_sweep_dev(N, n, d):
    q, r = divmod(N, n)
    lo = d * q + min(d, r)
    hi = (d + 1) * q + min(d + 1, r)
    i0, i1 = max(lo, 1), min(hi, N - 1)
    if i1 <= i0:
        return 0
    return 8 * N * (i1 - i0 + 2) + 8 * (i1 - i0) * (N - 2)


def _time_loop(J, C, fn, reps):
    """Device time per call (max over devices/ranks) of fn, plus the
    profiled average kernel and merge time per launch on device 0."""
    fn()
    J.jacc_set_profiling(1)
    J.jacc_profile_reset()
    t = C.timed(fn, reps) / reps
    k, m, nl, _ = J.jacc_profile_totals(C.local[0])
    J.jacc_set_profiling(0)
    return t, k / max(nl, 1), m / max(nl, 1)


def run_extra_loops(J, C, n, peak):
    """The other BASELINE configs (DOT 2^30, GEMM 8192^3, SCAT 2^28) timed
    through the same C-ABI: kernel-level roofline evidence, not bench lines."""
    import synth
    out = {}
    IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT
    # DOT 2^30
    L = 2**30
    x = synth.uniform_f64(L, 1, synth.AID["x"])
    y = synth.uniform_f64(L, 1, synth.AID["y"])
    s = np.zeros(1)
    for a in (x, y):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    dargs = [J.arg(IN, x), J.arg(IN, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)]
    rng = J.make_range(0, L)
    t, k, _ = _time_loop(J, C, lambda: J.jacc_launch(J.JACC_LOOP_DOT_F64, rng, dargs), 10)
    byts = 16 * L
    out["dot_2^30"] = {"loop_gbs": byts / t / 1e9, "kernel_us": k * 1e6,
                       "kernel_gbs": byts / n / k / 1e9, "frac_of_peak": byts / n / k / 1e9 / peak,
                       "frac_of_spec": byts / n / k / 1e9 / HBM_SPEC_GBS,
                       "launch_ms": t * 1e3}
    J.jacc_data_delete(x)
    J.jacc_data_delete(y)
    del x, y
    # GEMM 8192^3
    G = 8192
    Ag = synth.uniform_f64(G * G, 2, synth.AID["A"]).reshape(G, G)
    Bg = synth.uniform_f64(G * G, 2, synth.AID["B"]).reshape(G, G)
    Cg = np.zeros((G, G))
    for a in (Ag, Bg, Cg):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    gargs = [J.arg(IN, Ag), J.arg(IN, Bg), J.arg(OUT, Cg)]
    t, k, m = _time_loop(J, C, lambda: J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, gargs, 0), 3)
    fl = 2 * G**3
    dg, dsrc = load_dgemm_peak()
    out["gemm_8192"] = {"loop_tflops": fl / t / 1e12, "kernel_ms": k * 1e3,
                        "kernel_tflops": fl / n / k / 1e12, "merge_ms": m * 1e3,
                        "frac_of_cublas_dgemm": fl / n / k / 1e12 / dg if dg else None,
                        "cublas_dgemm_tflops": dg, "cublas_source": dsrc,
                        "frac_of_spec": fl / n / k / 1e12 / FP64_SPEC_TFLOPS,
                        "launch_ms": t * 1e3}
    for a in (Ag, Bg, Cg):
        J.jacc_data_delete(a)
    del Ag, Bg, Cg
    # SCAT 2^28 f64
    S = 2**28
    idx = synth.index_i32(S, S, 3, synth.AID["idx"])
    b = synth.dyadic_f64(S, 3, synth.AID["b"])
    a = synth.dyadic_f64(S, 3, synth.AID["a0"])
    for arr in (idx, b, a):
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    sargs = [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)]
    srng = J.make_range(0, S)
    t, k, m = _time_loop(J, C,
                         lambda: J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, srng, sargs, 0), 5)
    byts = S * (4 + 8 + 16)
    out["scatter_f64_2^28"] = {"loop_gbs": byts / t / 1e9, "kernel_us": k * 1e6,
                               "kernel_alg_gbs": byts / k / 1e9 if n == 1 else None,
                               "frac_of_peak": byts / k / 1e9 / peak if n == 1 else None,
                               "frac_of_spec": byts / k / 1e9 / HBM_SPEC_GBS if n == 1 else None,
                               # sector-level floor: 32 B read + 32 B write of a per update
                               "frac_of_sector_roofline": S * (4 + 8 + 64) / k / 1e9 / peak if n == 1 else None,
                               "merge_us": m * 1e6, "launch_ms": t * 1e3}
    for arr in (idx, b, a):
        J.jacc_data_delete(arr)
    del idx, b, a
    # Himeno XL (NEXT-2 workload): stencil + gosa, then copy, fp32
    I, Jd, K = 1025, 513, 513
    hp, ha, hb, hc, hw1, hbd = synth.himeno_init(I, Jd, K)
    hw2 = np.zeros_like(hp)
    for arr in (hp, ha, hb, hc, hw1, hbd, hw2):
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    g = np.zeros(1)
    hargs = [J.arg(IN, hp), J.arg(IN, ha), J.arg(IN, hb), J.arg(IN, hc), J.arg(IN, hw1),
             J.arg(IN, hbd), J.arg(OUT, hw2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
             J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)]
    cargs = [J.arg(IN, hw2), J.arg(OUT, hp)]
    ts, ks, _ = _time_loop(J, C, lambda: J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None, hargs, 0), 5)
    tc, kc, _ = _time_loop(J, C, lambda: J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None, cargs, 0), 5)
    pts = (I - 2) * (Jd - 2) * (K - 2)
    sb, cb = 56 * pts, 8 * pts   # 12 coefficient/aux arrays + p read, wrk2 written | copy
    out["himeno_XL_fp32"] = {"stencil_us": ks * 1e6, "stencil_gbs": sb / n / ks / 1e9,
                             "stencil_frac": sb / n / ks / 1e9 / peak,
                             "stencil_frac_of_spec": sb / n / ks / 1e9 / HBM_SPEC_GBS,
                             "copy_us": kc * 1e6, "copy_gbs": cb / n / kc / 1e9,
                             "iteration_ms": (ts + tc) * 1e3, "gosa": float(g[0])}
    for arr in (hp, ha, hb, hc, hw1, hbd, hw2):
        J.jacc_data_delete(arr)
    return out


def eager_merge_probe(J, torch, A, B):
    """BK5 merge kernel bandwidth: J16K with two virtual devices on this GPU
    under EAGER, so after every launch each device pushes its ~1 GiB dirty
    half into the other replica.  On one GPU the push is a local HBM copy
    (read + write), a proxy for the kernel's efficiency, not NVLink."""
    J.jacc_init(2, [0, 0])
    J.jacc_set_merge_policy(J.JACC_MERGE_EAGER)
    for arr in (A, B):
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    args_ab = [J.arg(IN, A), J.arg(OUT, B)]
    J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, args_ab, 0)
    J.jacc_wait()
    J.jacc_set_profiling(1)
    J.jacc_profile_reset()
    reps = 6
    for _ in range(reps):
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, args_ab, 0)
    J.jacc_wait()
    k, m, nl, _ = J.jacc_profile_totals(0)
    J.jacc_set_profiling(0)
    lo, hi = J.jacc_partition(N_GRID, 2, 0)
    dirty_bytes = (min(hi, N_GRID - 1) - max(lo, 1)) * N_GRID * 8   # span rows x full width
    J.jacc_finalize()
    mt = m / max(nl, 1)
    return {"merge_us": mt * 1e6, "bytes_pushed": dirty_bytes,
            "copy_gbs": 2 * dirty_bytes / mt / 1e9,
            "note": "one peer, virtual devices: local HBM read+write, not NVLink"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="jacc", choices=["jacc", "reference"])
    ap.add_argument("--merge", default="halo", choices=["halo", "eager"])
    ap.add_argument("--no-extra", dest="extra", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-sweeps", type=int, default=10)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_jacc(args)


if __name__ == "__main__":
    main()
