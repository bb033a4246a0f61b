"""Division of multidimensional arrays (Sec 4.2) written
out plainly -- TEST INFRASTRUCTURE ONLY (oracle for libjacc's
jacc_select_split_dim / jacc_exchange_plan and the strided merges).

  P:524-525 "we select the parallel dimension for each updated array to
            have the most parallel iterators while containing the least
            sequential iterators ... When there are several candidates, we
            choose the leftmost dimension in the C language and the
            rightmost dimension in Fortran"
  P:527     "Each kernel execution is performed while equally dividing
            parallel dimensions among GPUs and accompanied by the
            GPU-to-GPU communication through cudaMemcpy2DAsync."
Small cases only (pure-Python loops).
"""
from . import partition


def select_split_dim(n_parallel, n_sequential, fortran=False):
    """Return the split dimension, or -1 (duplicate) if no dimension holds
    a parallel iterator.  Candidates: most parallel iterators; among them
    the fewest sequential iterators; ties: leftmost (C) / rightmost."""
    nd = len(n_parallel)
    best = max(n_parallel) if nd else 0
    if best == 0:
        return -1
    cands = [k for k in range(nd) if n_parallel[k] == best]
    fewest = min(n_sequential[k] for k in cands)
    cands = [k for k in cands if n_sequential[k] == fewest]
    return cands[-1] if fortran else cands[0]


def slice_elements(extents, split_dim, lo, hi):
    """Sorted flat (row-major) indices of every element whose index along
    split_dim lies in [lo, hi): the device's owned slice, enumerated by
    brute force over all elements."""
    out = []
    total = 1
    for e in extents:
        total *= e
    for f in range(total):
        rem, idx = f, []
        for e in reversed(extents):
            idx.append(rem % e)
            rem //= e
        idx.reverse()
        if lo <= idx[split_dim] < hi:
            out.append(f)
    return out


def owned_block(extents, split_dim, n, d):
    return partition(extents[split_dim], n, d)
