"""N>1 launch contract on CPU (gloo, world size 2): the reference arm of
bench.py under torch.distributed.run prints exactly one JSON line from
rank 0 and every rank exits 0."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_reference_arm_torchrun_world2():
    env = dict(os.environ, JACC_BENCH_REF_SWEEPS="1", JACC_BENCH_REF_N="2048")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "oracle"


def test_blob_exchange_plumbing_world2(tmp_path):
    """The bootstrap collectives of paper_2110_14340_b200.dist move opaque
    blobs between 2 gloo ranks (no GPU needed for the transport itself)."""
    script = tmp_path / "w.py"
    script.write_text(
        "import sys, torch.distributed as dist\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "dist.init_process_group('gloo')\n"
        "r = dist.get_rank()\n"
        "from paper_2110_14340_b200 import dist as jd\n"
        "got = jd._all_gather(bytes([r]) * 64)\n"
        "assert got == [bytes([0]) * 64, bytes([1]) * 64], got\n"
        "dist.destroy_process_group()\n")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
