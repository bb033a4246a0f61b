"""bench.py -- headline benchmark of the JACC B200 hot path.

Workload (BASELINE.json configs[1]): Jacobi-2D fp64 16384 x 16384, 100
timesteps = 200 `parallel loop` launches per step, owned row blocks over N
devices with HALO (boundary-row dirty-range) merge.  Metric: algorithmic
loop GB/s (8 B read per src element + 8 B written per interior dst element
per launch), whole job.  Inputs (2 x 2 GiB) are far larger than L2, so no
explicit flush is needed between timed iterations.

The other BASELINE configs (DOT 2^30, GEMM 8192^3, SCAT 2^28 f64 and i32)
and the Himeno XL workload are measured in the same run under "loops", each
with its own roofline block, CPU-oracle baseline and end-to-end number; the
BK5 merge kernels are measured in isolation under "merge".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl jacc|reference]

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (the
only reference this tier has) on a bounded sample of the same workload,
pinned to one host core.
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
WORKLOAD = "J16K: Jacobi-2D fp64 16384x16384, 100 timesteps (200 launches/step)"

HBM_SPEC_GBS = 8000.0      # B200 datasheet HBM3e
FP64_SPEC_TFLOPS = 40.0    # B200 datasheet fp64 (tensor), SURVEY 8(d)
NVLINK_GBS = 770.0         # measured peer copy per direction (B200_PROFILING.md); 900 nominal
NVLINK_SPEC_GBS = 900.0
FP64_PER_BF16 = 40.0 / 2250.0   # nominal fp64 tensor / dense bf16 ratio (guide)

# workload sizes (BASELINE.json configs)
DOT_L = 2**30
GEMM_N = 8192
SCAT_N = 2**28
HIMENO = (1024, 512, 512)  # Size XL grid (DESIGN R-17)


def algo_bytes_per_sweep_dev(N, n, d):
    """Algorithmic HBM bytes of one Jacobi launch on device d: its owned rows
    plus one halo row each side read (8 B/element), its interior elements
    written (8 B/element)."""
    q, r = divmod(N, n)
    lo = d * q + min(d, r)
    hi = (d + 1) * q + min(d + 1, r)
    i0, i1 = max(lo, 1), min(hi, N - 1)
    if i1 <= i0:
        return 0
    return 8 * N * (i1 - i0 + 2) + 8 * (i1 - i0) * (N - 2)


def algo_bytes_per_sweep(N, n):
    return sum(algo_bytes_per_sweep_dev(N, n, d) for d in range(n))


def halo_bytes_dev(N, n, d):
    """Bytes device d pushes per Jacobi launch under HALO: its first and last
    interior rows (N-2 doubles each) to the neighbours that read them."""
    if n == 1:
        return 0
    q, r = divmod(N, n)
    lo = d * q + min(d, r)
    hi = (d + 1) * q + min(d + 1, r)
    if min(hi, N - 1) <= max(lo, 1):
        return 0
    rows = (1 if d > 0 else 0) + (1 if d < n - 1 else 0)
    return rows * 8 * (N - 2)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


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


def load_traffic(*kernels):
    """DRAM bytes (read + write) per launch summed over the given kernels,
    from the newest committed ncu --set full summary (profiles/), or None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")), reverse=True):
        try:
            with open(p) as f:
                j = json.load(f).get("kernels", {})
            if all(j.get(k, {}).get("dram_bytes_per_launch") for k in kernels):
                return sum(float(j[k]["dram_bytes_per_launch"]) for k in kernels), os.path.basename(p)
        except Exception:
            pass
    return None, None


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, cuda_ords):
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
        never leaves the timed region unsampled"""
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
            if not inside:
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
# CPU oracle timing (cpu_baseline leg and the reference arm).  Runs in a child
# process pinned to ONE host core (sched_setaffinity == taskset -c), on the
# same seeded inputs as the GPU run (synth/), each a bounded sample.
# ----------------------------------------------------------------------------
def _oracle_worker(name, arg):
    core = sorted(os.sched_getaffinity(0))[-1]
    os.sched_setaffinity(0, {core})
    import __graft_entry__ as ge
    ge.build_oracle()
    ge.build_synth()
    import oracle as orc
    import synth
    res = {"core": core}
    if name == "j16k":
        sweeps = int(arg)
        A, B = synth.polybench_jacobi2d(N_GRID)
        t0 = time.perf_counter()
        src, dst = A, B
        for _ in range(sweeps):
            orc.jacobi2d_sweep(src, dst)
            src, dst = dst, src
        dt = time.perf_counter() - t0
        res.update(seconds=dt, work=sweeps * algo_bytes_per_sweep(N_GRID, 1),
                   sample=f"{sweeps} oracle sweeps of the 16384^2 grid (of 200 per step)")
    elif name == "dot":
        L = int(arg)
        x = synth.uniform_f64(L, 1, synth.AID["x"])
        y = synth.uniform_f64(L, 1, synth.AID["y"])
        t0 = time.perf_counter()
        orc.dot_f64(x, y, 0.0)
        dt = time.perf_counter() - t0
        res.update(seconds=dt, work=16 * L,
                   sample=f"oracle dot over the first {L} of the 2^30 elements (same seeded x, y)")
    elif name == "gemm":
        rows = int(arg)
        G = GEMM_N
        A = synth.uniform_f64(G * G, 2, synth.AID["A"]).reshape(G, G)
        B = synth.uniform_f64(G * G, 2, synth.AID["B"]).reshape(G, G)
        Ar = np.ascontiguousarray(A[:rows])
        t0 = time.perf_counter()
        orc.gemm_f64(Ar, B, ikj=True)
        dt = time.perf_counter() - t0
        res.update(seconds=dt, work=2 * rows * G * G,
                   sample=f"oracle GEMM (i-k-j form, bit-identical to i-j-k, DESIGN R-11) of C rows "
                          f"[0, {rows}) of 8192 (same A, B); "
                          f"rate scales linearly to the full product")
    elif name in ("scat_f64", "scat_i32"):
        n_upd = int(arg)
        idx = synth.index_i32(SCAT_N, SCAT_N, 3, synth.AID["idx"])[:n_upd].copy()
        if name == "scat_f64":
            b = synth.dyadic_f64(SCAT_N, 3, synth.AID["b"])[:n_upd].copy()
            a = synth.dyadic_f64(SCAT_N, 3, synth.AID["a0"])
            per = 28
        else:
            b = synth.int_i32(SCAT_N, -1000, 1000, 3, synth.AID["b"])[:n_upd].copy()
            a = synth.int_i32(SCAT_N, -10**6, 10**6, 3, synth.AID["a0"])
            per = 16
        t0 = time.perf_counter()
        orc.scatter_add(idx, b, a)
        dt = time.perf_counter() - t0
        res.update(seconds=dt, work=per * n_upd,
                   sample=f"oracle a[idx[i]] += b[i] for the first {n_upd} of the 2^28 updates "
                          f"into the full 2^28-element a (same seeded idx, b, a)")
    else:
        raise SystemExit(f"unknown oracle worker {name}")
    print(json.dumps(res), flush=True)


def cpu_baseline(name, arg, unit, scale):
    """Run the oracle worker in a child pinned to one core; value = work /
    seconds * scale in `unit`."""
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-worker", name,
                        "--oracle-arg", str(arg)], capture_output=True, text=True, cwd=ROOT)
    if r.returncode != 0:
        return {"value": None, "unit": unit, "error": r.stderr.strip()[-300:]}
    j = json.loads(r.stdout.strip().splitlines()[-1])
    hi = host_info()
    return {"value": j["work"] / j["seconds"] * scale, "unit": unit, "cores": 1, "kind": "oracle",
            "sample": j["sample"], "seconds": j["seconds"], "pinned_core": j["core"],
            "host_nproc": hi["nproc"], "host_model": hi["model"],
            "oracle": "oracle/oracle.c, gcc -O2 -ffp-contract=off, single thread"}


def run_reference(args):
    """The reference arm of this tier: the CPU oracle on a bounded sample of
    the J16K step (2 of its 200 sweeps per timed step), pinned to one core.
    ms_per_step and value are what was timed (no extrapolation)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sweeps = 2
    for _ in range(args.warmup):
        cpu_baseline("j16k", 1, UNIT, 1e-9)
    vals, times, last = [], [], None
    for _ in range(args.steps):
        last = cpu_baseline("j16k", sweeps, UNIT, 1e-9)
        vals.append(last["value"])
        times.append(last["seconds"])
    v = statistics.median(vals)
    cb = dict(last)
    cb["value"] = v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3, "extrapolated": False,
        "step": f"one step = {sweeps} of the 200 oracle sweeps of a J16K step (bounded sample)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (PolyBench jacobi-2d init)",
        "config": {"workload": WORKLOAD, "sample": cb.get("sample"),
                   "l2": "inputs 2x2 GiB >> 126 MB L2"},
        "cpu_baseline": cb,
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
    info = J.jacc_get_info()
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
        timed_step = lambda: J.jacc_graph_replay(gid, 1)  # noqa: E731
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
    peaks, peak_src = load_peaks()
    peak = float(peaks["hbm_gbs"])
    traffic, tsrc = load_traffic("jacobi2d")
    if traffic is not None and n > 1:
        traffic = None  # the committed capture is of the n=1 launch
    # two-term per-launch roofline: the
    # slower of the busiest device's HBM bytes and its merged bytes over
    # NVLink (HALO: two boundary rows per interior device per launch)
    merged_dev = max(halo_bytes_dev(N, n, d) for d in range(n)) if args.merge == "halo" else \
        max((algo_bytes_per_sweep_dev(N, n, d) // 2) * (n - 1) for d in range(n)) if n > 1 else 0
    t_hbm = max(algo_bytes_per_sweep_dev(N, n, d) for d in range(n)) / (peak * 1e9)
    t_nvl = merged_dev / (NVLINK_GBS * 1e9)
    t_roof = max(t_hbm, t_nvl)
    t_launch = t / args.steps / (2 * TSTEPS)

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
    e2e_h2d, e2e_d2h = A.nbytes + B.nbytes, A.nbytes

    loops, merge = {}, {}
    if args.extra and not C.mp:
        J.jacc_data_delete(A)
        J.jacc_data_delete(B)
        loops = run_loops(J, C, n, peaks, args)
    C.finalize()
    if args.extra and not C.mp and n == 1:
        del A, B
        merge = merge_probes(J)

    cpu = None
    if args.cpu_baseline and n == 1 and C.rank == 0:
        cpu = cpu_baseline("j16k", args.cpu_sweeps, UNIT, 1e-9)
        for name, (key, arg, unit, scale) in {
                "dot_2^30": ("dot", 2**29, "GB/s", 1e-9),
                "gemm_8192": ("gemm", 32, "TFLOP/s", 1e-12),
                "scatter_f64_2^28": ("scat_f64", 2**26, "GB/s", 1e-9),
                "scatter_i32_2^28": ("scat_i32", 2**26, "GB/s", 1e-9)}.items():
            if name in loops:
                loops[name]["cpu_baseline"] = cpu_baseline(key, arg, unit, scale)
    if C.rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (PolyBench jacobi-2d init, seeded generators in synth/)",
        "config": {"workload": WORKLOAD,
                   "merge": args.merge, "launch": "one process per GPU" if C.mp else "single process",
                   "issue": "CUDA graph replay of the captured step" if use_graph else "jacc_launch x200",
                   "ms_per_step_plain_launches": t_plain * 1e3,
                   "host_us_per_launch": host_us,
                   "virtual_devices": C.virtual,
                   "combine": info["combine"], "distinct_gpus": bool(info["distinct_gpus"]),
                   "peer_pairs": info["peer_pairs"],
                   "l2": "no flush: inputs 2x2 GiB >> 126 MB L2",
                   "parallelism": f"row-block owner partition over {n} device(s)"},
        "roofline": {"bound": "hbm" if t_hbm >= t_nvl else "nvlink", "achieved": achieved,
                     "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "frac_of_spec": achieved / HBM_SPEC_GBS, "spec_peak": HBM_SPEC_GBS,
                     "kernel": "jacobi2d_kernel", "kernel_avg_us": k_avg * 1e6,
                     "algo_bytes_per_launch": per_dev_bytes, "peak_source": peak_src,
                     "traffic_source": tsrc,
                     "two_term": {"merged_bytes_per_device_per_launch": merged_dev,
                                  "nvlink_gbs": NVLINK_GBS, "nvlink_spec_gbs": NVLINK_SPEC_GBS,
                                  "t_hbm_us": t_hbm * 1e6, "t_nvlink_us": t_nvl * 1e6,
                                  "t_roof_us": t_roof * 1e6, "t_launch_us": t_launch * 1e6,
                                  "frac_of_t_roof": t_roof / t_launch if t_launch else None}},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": e2e_h2d,
                "d2h_bytes_per_step": e2e_d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "host": host_info(),
    }
    if loops:
        line["loops"] = loops
    if merge:
        line["merge"] = merge
    print(json.dumps(line), flush=True)


def _time_loop(J, C, fn, reps):
    """Device time per call (max over devices/ranks) of fn, plus the
    profiled average kernel and merge time per launch on device 0."""
    fn()
    J.jacc_wait()
    J.jacc_set_profiling(1)
    J.jacc_profile_reset()
    t = C.timed(fn, reps) / reps
    k, m, nl, _ = J.jacc_profile_totals(C.local[0])
    J.jacc_set_profiling(0)
    return t, k / max(nl, 1), m / max(nl, 1)


def _e2e(J, C, upload, launch, download, reps=2):
    """Seconds per end-to-end call through the public API: H2D of the
    inputs from the (pinned) host arrays, the launch, D2H of the result."""
    ts = []
    for it in range(reps + 1):
        C.sync()
        t0 = time.perf_counter()
        for a in upload:
            J.jacc_update_device(a)
        launch()
        for a in download:
            J.jacc_update_host(a)
        J.jacc_wait()
        if it:
            ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def _hbm_roof(achieved, peak, peak_src, kernels, algo, k, traffic_keys):
    traffic, tsrc = load_traffic(*traffic_keys)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
            "frac_of_spec": achieved / HBM_SPEC_GBS, "spec_peak": HBM_SPEC_GBS,
            "kernel": kernels, "kernel_avg_us": k * 1e6, "algo_bytes_per_launch": algo,
            "peak_source": peak_src}


def cublas_dgemm_tflops(torch, A, B, reps=5):
    """cuBLAS DGEMM (torch.matmul on fp64 device tensors) on the same inputs:
    the measured fp64 tensor-pipe reference for the GEMM roofline (a library
    GEMM used as the denominator only, never on the product path)."""
    try:
        a = torch.from_numpy(A).cuda()
        b = torch.from_numpy(B).cuda()
        torch.matmul(a, b)
        torch.cuda.synchronize()
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None or t < best else best
        del a, b
        torch.cuda.empty_cache()
        return 2 * A.shape[0] * A.shape[1] * B.shape[1] / best / 1e12
    except Exception:
        return None


def run_loops(J, C, n, peaks, args):
    """The other BASELINE configs (DOT 2^30, GEMM 8192^3, SCAT 2^28 f64 and
    int32) and Himeno XL, timed through the same C-ABI.  Each entry carries
    its metric, roofline block (algorithmic bytes or FLOPs / CUDA-event
    kernel time vs the measured peak, ncu DRAM bytes), e2e through the
    public API with declared bytes, and (n = 1) a CPU-oracle baseline."""
    import synth
    peak = float(peaks["hbm_gbs"])
    psrc = "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    out = {}
    IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT
    # ---- DOT 2^30 (uniform [0,1), tolerance config) ----
    L = DOT_L
    x = synth.uniform_f64(L, 1, synth.AID["x"])
    y = synth.uniform_f64(L, 1, synth.AID["y"])
    s = np.zeros(1)
    for a in (x, y):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    dargs = [J.arg(IN, x), J.arg(IN, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)]
    rng = J.make_range(0, L)
    launch = lambda: J.jacc_launch(J.JACC_LOOP_DOT_F64, rng, dargs)  # noqa: E731
    t, k, _ = _time_loop(J, C, launch, 10)
    byts = 16 * L
    te = _e2e(J, C, [x, y], launch, [])
    out["dot_2^30"] = {
        "workload": "DOT: s += x[i]*y[i], fp64, 2^30 elements, uniform [0,1)",
        "metric": "loop GB/s", "value": byts / t / 1e9, "unit": "GB/s", "launch_ms": t * 1e3,
        "roofline": _hbm_roof(byts / n / k / 1e9, peak, psrc, "reduce_kernel", byts // n, k, ["dot"]),
        "e2e": {"value": byts / te / 1e9, "unit": "GB/s", "seconds": te,
                "h2d_bytes_per_step": x.nbytes + y.nbytes, "d2h_bytes_per_step": 8},
    }
    J.jacc_data_delete(x)
    J.jacc_data_delete(y)
    del x, y
    # ---- GEMM 8192^3 ----
    G = GEMM_N
    Ag = synth.uniform_f64(G * G, 2, synth.AID["A"]).reshape(G, G)
    Bg = synth.uniform_f64(G * G, 2, synth.AID["B"]).reshape(G, G)
    Cg = np.zeros((G, G))
    for a in (Ag, Bg, Cg):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    gargs = [J.arg(IN, Ag), J.arg(IN, Bg), J.arg(OUT, Cg)]
    launch = lambda: J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, gargs, 0)  # noqa: E731
    t, k, m = _time_loop(J, C, launch, 3)
    fl = 2 * G**3
    dg, dsrc = load_dgemm_peak()
    dg_run = cublas_dgemm_tflops(C.torch, Ag, Bg)  # same box, same run: the fp64 reference
    if dg_run:
        dg, dsrc = dg_run, "torch.matmul fp64 (cuBLAS DGEMM) 8192^3 timed in this run"
    scaled = float(peaks.get("bf16_tflops", 0)) * FP64_PER_BF16
    te = _e2e(J, C, [Ag, Bg], launch, [Cg], reps=1)
    traffic, tsrc = load_traffic("gemm")
    ach = fl / n / k / 1e12
    pk = dg if dg else scaled
    out["gemm_8192"] = {
        "workload": "GEMM: C = A B, fp64 8192^3, uniform [0,1), row blocks of C",
        "metric": "loop TFLOP/s", "value": fl / t / 1e12, "unit": "TFLOP/s", "launch_ms": t * 1e3,
        "merge_ms": m * 1e3,
        "roofline": {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                     "frac": ach / pk, "traffic": traffic, "traffic_source": tsrc,
                     "peak_source": (f"cuBLAS DGEMM 8192^3: {dsrc}" if dg
                                     else "MEASURED_PEAKS bf16 burst x nominal fp64/bf16 ratio"),
                     "peak_bf16_scaled": scaled, "frac_of_bf16_scaled": ach / scaled if scaled else None,
                     "spec_peak": FP64_SPEC_TFLOPS, "frac_of_spec": ach / FP64_SPEC_TFLOPS,
                     "kernel": "gemm_tma_kernel (TMA + mbarrier ring, DMMA)", "kernel_avg_ms": k * 1e3,
                     "algo_flops_per_launch": fl // n},
        "e2e": {"value": fl / te / 1e12, "unit": "TFLOP/s", "seconds": te,
                "h2d_bytes_per_step": Ag.nbytes + Bg.nbytes, "d2h_bytes_per_step": Cg.nbytes},
    }
    for a in (Ag, Bg, Cg):
        J.jacc_data_delete(a)
    del Ag, Bg, Cg
    # ---- SCAT 2^28 (f64 dyadic, int32) ----
    S = SCAT_N
    idx = synth.index_i32(S, S, 3, synth.AID["idx"])
    for dt in ("f64", "i32"):
        if dt == "f64":
            b = synth.dyadic_f64(S, 3, synth.AID["b"])
            a = synth.dyadic_f64(S, 3, synth.AID["a0"])
            loop, per = J.JACC_LOOP_SCATTER_ADD_F64, 28
        else:
            b = synth.int_i32(S, -1000, 1000, 3, synth.AID["b"])
            a = synth.int_i32(S, -10**6, 10**6, 3, synth.AID["a0"])
            loop, per = J.JACC_LOOP_SCATTER_ADD_I32, 16
        for arr in (idx, b, a):
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        sargs = [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)]
        srng = J.make_range(0, S)
        launch = lambda: J.jacc_launch(loop, srng, sargs, 0)  # noqa: E731
        t, k, m = _time_loop(J, C, launch, 5)
        byts = S * per
        te = _e2e(J, C, [idx, b, a], launch, [a], reps=1)
        tk = [f"scat_{p}" + ("" if dt == "f64" else "_i32") for p in ("part", "apply", "bits")]
        ach = byts / k / 1e9 if n == 1 else None
        out[f"scatter_{dt}_2^28"] = {
            "workload": f"SCAT: a[idx[i]] += b[i], {dt}, 2^28 updates into 2^28 elements, "
                        "idx uniform random (63% distinct targets)",
            "metric": "loop GB/s", "value": byts / t / 1e9, "unit": "GB/s", "launch_ms": t * 1e3,
            "merge_us": m * 1e6,
            "roofline": _hbm_roof(ach, peak, psrc, "binned scatter pipeline (all kernels of the launch)",
                                  byts, k, tk) if n == 1 else None,
            "e2e": {"value": byts / te / 1e9, "unit": "GB/s", "seconds": te,
                    "h2d_bytes_per_step": idx.nbytes + b.nbytes + a.nbytes,
                    "d2h_bytes_per_step": a.nbytes},
        }
        for arr in (idx, b, a):
            J.jacc_data_delete(arr)
        del b, a
    del idx
    # ---- Himeno XL (NEXT-2 workload): stencil + gosa, then copy, fp32 ----
    I, Jd, K = HIMENO
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
    out["himeno_XL_fp32"] = {
        "workload": f"Himeno {I}x{Jd}x{K} fp32: 19-point stencil + gosa, then copy",
        "metric": "loop GB/s", "value": (sb + cb) / (ts + tc) / 1e9, "unit": "GB/s",
        "iteration_ms": (ts + tc) * 1e3, "gosa": float(g[0]),
        "roofline": _hbm_roof(sb / n / ks / 1e9, peak, psrc, "himeno_stencil_kernel", sb // n, ks,
                              ["himeno_stencil"]),
        "copy": {"us": kc * 1e6, "gbs": cb / n / kc / 1e9, "frac": cb / n / kc / 1e9 / peak},
    }
    for arr in (hp, ha, hb, hc, hw1, hbd, hw2):
        J.jacc_data_delete(arr)
    return out


def merge_probes(J):
    """BK5 merge kernels in isolation: two logical
    devices on this GPU under EAGER, with the loop restricted to device 0's
    block so device 1 runs no loop kernel and device 0's merge is the only
    work in flight.  On one GPU the peer replica is local HBM, so the merge
    is an HBM read + write: its fraction of the copy peak is the kernel's
    efficiency; on distinct GPUs the same kernel's stores cross NVLink."""
    import synth
    peaks, _ = load_peaks()
    peak = float(peaks["hbm_gbs"])
    out = {}
    IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT

    def prof(fn, reps):
        fn()
        J.jacc_wait()
        J.jacc_set_profiling(1)
        J.jacc_profile_reset()
        for _ in range(reps):
            fn()
        J.jacc_wait()
        k, m, nl, _ = J.jacc_profile_totals(0)
        J.jacc_set_profiling(0)
        return m / max(nl, 1)

    # merge_range: Jacobi rows [1, 8192) = device 0's block (device 1 idle)
    J.jacc_init(2, [0, 0])
    try:
        J.jacc_set_merge_policy(J.JACC_MERGE_EAGER)
        N = N_GRID
        A, B = synth.polybench_jacobi2d(N)
        for arr in (A, B):
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        lo, hi = J.jacc_partition(N, 2, 0)
        rng = J.make_range((lo + 1, 1), (hi, N - 1))
        args_ab = [J.arg(IN, A), J.arg(OUT, B)]
        mt = prof(lambda: J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, rng, args_ab, 0), 6)
        span = ((hi - 1) * N + N - 2) - ((lo + 1) * N + 1) + 1
        byts = 8 * span
        out["merge_range"] = {"kernel": "merge_range_bulk_kernel", "us": mt * 1e6,
                              "dirty_bytes": byts, "copy_gbs": 2 * byts / mt / 1e9,
                              "frac_of_hbm_copy": 2 * byts / mt / 1e9 / peak,
                              "nvlink_time_at_770_us": byts / (NVLINK_GBS * 1e9) * 1e6}
        del A, B
    finally:
        J.jacc_finalize()
    # merge_bitmap: scatter whose targets all fall in device 0's slice, with
    # the direct scatter kernel (the binned pipeline fuses the push into its
    # bits pass, measured below)
    M = SCAT_N
    os.environ["JACC_SCATTER_BINNED"] = "0"
    for name, nupd in (("merge_bitmap_dense", 2**27), ("merge_bitmap_sparse", 2**20)):
        J.jacc_init(2, [0, 0])
        try:
            J.jacc_set_merge_policy(J.JACC_MERGE_EAGER)
            idx = synth.index_i32(nupd, M // 2, 4, synth.AID["idx"])
            b = synth.dyadic_f64(nupd, 4, synth.AID["b"])
            a = synth.dyadic_f64(M, 4, synth.AID["a0"])
            for arr in (idx, b, a):
                J.jacc_data_create(arr)
                J.jacc_update_device(arr)
            sargs = [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)]
            mt = prof(lambda: J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(0, nupd),
                                            sargs, 0), 4)
            bm = J.jacc_get_dirty_bitmap(a, 0, M)
            dirty = int(np.unpackbits(bm.view(np.uint8)).sum())
            words = (M // 2 + 31) // 32
            moved = 8 * _pushed_elements(bm, 0, M // 2)
            out[name] = {"kernel": "merge_bitmap_kernel", "us": mt * 1e6, "updates": nupd,
                         "dirty_elements": dirty, "bitmap_words_scanned": words,
                         "bytes_pushed": moved, "dense_word_rule": DENSE_RULE,
                         "hbm_bytes": 2 * moved + 4 * words,
                         "gbs": (2 * moved + 4 * words) / mt / 1e9,
                         "frac_of_hbm_copy": (2 * moved + 4 * words) / mt / 1e9 / peak,
                         "nvlink_time_at_770_us": moved / (NVLINK_GBS * 1e9) * 1e6}
            del idx, b, a
        finally:
            J.jacc_finalize()
    del os.environ["JACC_SCATTER_BINNED"]
    # binned scatter under EAGER: device 0's launch time (binned pipeline +
    # merge_bitmap of its dirty words into the peer) minus the same launch
    # under HALO (no push)
    J.jacc_init(2, [0, 0])
    try:
        nupd = 2**27
        idx = synth.index_i32(nupd, M // 2, 4, synth.AID["idx"])
        b = synth.dyadic_f64(nupd, 4, synth.AID["b"])
        a = synth.dyadic_f64(M, 4, synth.AID["a0"])
        for arr in (idx, b, a):
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        sargs = [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)]
        tk = {}
        for pol in (J.JACC_MERGE_HALO, J.JACC_MERGE_EAGER):
            J.jacc_set_merge_policy(pol)
            fn = lambda: J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(0, nupd), sargs, 0)  # noqa: E731
            fn()
            J.jacc_wait()
            J.jacc_set_profiling(1)
            J.jacc_profile_reset()
            for _ in range(4):
                fn()
            J.jacc_wait()
            k, m, nl, _ = J.jacc_profile_totals(0)
            J.jacc_set_profiling(0)
            tk[pol] = (k + m) / max(nl, 1)
        bm = J.jacc_get_dirty_bitmap(a, 0, M)
        moved = 8 * _pushed_elements(bm, 0, M // 2)
        extra = tk[J.JACC_MERGE_EAGER] - tk[J.JACC_MERGE_HALO]
        out["binned_scatter_eager_merge"] = {
            "kernel": "merge_bitmap_kernel after the binned scatter", "launch_us_halo": tk[J.JACC_MERGE_HALO] * 1e6,
            "launch_us_eager": tk[J.JACC_MERGE_EAGER] * 1e6, "push_cost_us": extra * 1e6,
            "bytes_pushed": moved, "push_gbs": 2 * moved / extra / 1e9 if extra > 0 else None,
            "merge_bitmap_dense_us": out.get("merge_bitmap_dense", {}).get("us"),
            "nvlink_time_at_770_us": moved / (NVLINK_GBS * 1e9) * 1e6}
        del idx, b, a
    finally:
        J.jacc_finalize()
    return out


DENSE_RULE = ("a bitmap word with >= 8 of its 32 elements dirty and inside the device's slice "
              "is pushed whole (kernels.cu merge_dense)")


def _pushed_elements(bm, lo, hi, dense_t=8):
    """Elements a bitmap merge stores into each peer for device slice [lo, hi):
    dense words whole, the others element by element (merge_dense)."""
    pop = np.unpackbits(bm.view(np.uint8)).reshape(-1, 32).sum(axis=1).astype(np.int64)
    w = np.arange(pop.size, dtype=np.int64)
    whole = (pop >= dense_t) & (w * 32 >= lo) & (w * 32 + 32 <= hi)
    return int(np.where(whole, 32, pop).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="jacc", choices=["jacc", "reference"])
    ap.add_argument("--merge", default="halo", choices=["halo", "eager"])
    ap.add_argument("--no-extra", dest="extra", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-sweeps", type=int, default=6)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--oracle-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--oracle-arg", default="1", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.oracle_worker:
        _oracle_worker(args.oracle_worker, args.oracle_arg)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_jacc(args)


if __name__ == "__main__":
    main()
