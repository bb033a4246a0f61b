"""Worker: randomised programs (tests/test_gpu_random_programs.Program) in
one-process-per-GPU mode.  Every rank runs the same seeds (SPMD); each
program starts a fresh runtime.  Prints "ok <count>" on success."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=20)
    ap.add_argument("--first", type=int, default=5000)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2110_14340_b200 import dist as jd
    from paper_2110_14340_b200 import jacc as J
    from test_gpu_random_programs import Program

    dist.init_process_group("gloo")
    ngpu = torch.cuda.device_count()
    ordinal = dist.get_rank() % ngpu
    torch.cuda.set_device(ordinal)
    for seed in range(a.first, a.first + a.seeds):
        _, world, _ = jd.init_rank(ordinal)
        try:
            Program(J, seed, world=world).run(40, jd.data_create)
        finally:
            jd.finalize()
    os.write(1, f"ok {a.seeds}\n".encode())  # one write: ranks share the pipe


if __name__ == "__main__":
    main()
