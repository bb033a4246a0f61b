"""One-off box probe: fp64 cuBLAS peak, HBM copy, host cores (context numbers for DESIGN.md)."""
import json, os, subprocess, time
import torch

out = {}
dev = torch.device("cuda:0")
p = torch.cuda.get_device_properties(0)
out["gpu"] = p.name
out["sms"] = p.multi_processor_count
out["mem_gb"] = p.total_memory / 1e9
out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
try:
    out["lscpu_model"] = [l for l in subprocess.check_output(["lscpu"], text=True).splitlines() if "Model name" in l][0]
except Exception as e:
    out["lscpu_model"] = str(e)

def t_ev(fn, reps):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

N = 8192
a = torch.rand(N, N, dtype=torch.float64, device=dev)
b = torch.rand(N, N, dtype=torch.float64, device=dev)
t = t_ev(lambda: torch.matmul(a, b), 5)
out["dgemm_8192_s"] = t
out["dgemm_tflops"] = 2 * N**3 / t / 1e12
del a, b
x = torch.empty(2**30, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
t = t_ev(lambda: y.copy_(x), 10)
out["copy_8GiB_gbs"] = 2 * x.numel() * 8 / t / 1e9
t = t_ev(lambda: torch.dot(x, y), 10)
out["torch_dot_2^30_gbs"] = 2 * x.numel() * 8 / t / 1e9
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
