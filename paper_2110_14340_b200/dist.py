"""One-process-per-GPU bootstrap over torch.distributed (plumbing only).

The C-ABI's multi-process mode (jacc_init_rank, include/jacc.h) needs a few
opaque byte blobs moved between ranks once: the NCCL unique id, the
shared-memory segment name, CUDA-IPC handles of every rank's events and
replicas.  This module moves them with torch.distributed object
collectives (gloo or nccl process group); no data-path bytes ever travel
through it -- merges, pulls and reductions run in libjacc's kernels, over
peer memory and NCCL.
"""
import os
import time

from . import jacc as J


def _world():
    import torch.distributed as dist
    return dist, dist.get_rank(), dist.get_world_size()


def _all_gather(obj):
    dist, _, world = _world()
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def init_rank(cuda_ordinal=None, use_nccl=None):
    """Collective: initialise this process as logical device `rank`."""
    import torch
    dist, rank, world = _world()
    if cuda_ordinal is None:
        cuda_ordinal = torch.cuda.current_device()
    uuid = str(torch.cuda.get_device_properties(cuda_ordinal).uuid)
    uuids = _all_gather(uuid)
    distinct = len(set(uuids)) == world
    if use_nccl is None:
        # JACC_NO_NCCL=1: the fixed-order peer-memory combine, explicitly
        use_nccl = distinct and world > 1 and not os.environ.get("JACC_NO_NCCL")
    if use_nccl and not distinct:
        raise ValueError("NCCL combine needs one distinct GPU per rank")
    box = [None]
    if rank == 0:
        box = [(J.jacc_unique_id() if use_nccl else None,
                f"jacc_{os.getpid()}_{time.time_ns()}")]
    dist.broadcast_object_list(box, src=0)
    uid, shm = box[0]
    J.jacc_init_rank(rank, world, cuda_ordinal, uid, shm)
    blobs = _all_gather(J.jacc_export_runtime())
    for peer, b in enumerate(blobs):
        if peer != rank:
            J.jacc_import_runtime(peer, b)
    dist.barrier()
    return rank, world, distinct


def data_create(arr):
    """Collective jacc_data_create + replica handle exchange."""
    _, rank, world = _world()
    J.jacc_data_create(arr)
    blobs = _all_gather(J.jacc_export_region(arr))
    for peer, b in enumerate(blobs):
        if peer != rank:
            J.jacc_import_region(arr, peer, b)


def finalize():
    dist, _, _ = _world()
    dist.barrier()
    J.jacc_finalize()
