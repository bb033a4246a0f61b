"""Automated asynchronous execution (Sec 3.2.1, Fig. 2)
written out plainly -- TEST INFRASTRUCTURE ONLY (oracle for libjacc's
jacc_queue_replay and the JACC_ASYNC_AUTO launch path).

  P:357-359 "Each JACC routine has the ability to track array references,
            and if data dependencies are encountered across two or more
            routines, JACC will schedule them in the same async queue."
  P:360-364 "When multiple queues are concerned, synchronous operations are
            performed only among those queues that require them, while
            skipping redundant synchronization on already solved
            dependencies. JACC achieves this by maintaining timestamps of
            data accesses and the most recent synchronization among queues."
  P:365     "If there is no data dependency to prior execution, the least
            recently used queue is selected."
  P:375-376 (Fig. 2) Kernel2 waits for the queues that updated a and b;
            "for Kernel3, the dependency on b is already solved by the
            previous synchronization, thus the execution does not wait".

Readings (DESIGN R-20): a dependency is RAW/WAW on the last writer of any
array the launch touches, or WAR on the last reader (per queue) of an array
it writes; with several dependencies the launch joins the queue of the most
recent one (ties: lowest queue index); a wait of queue q on queue p also
inherits everything p had synchronised with (transitive elision); the LRU
tie-break is the lowest queue index; an explicit queue (async(n)) is
honoured with the same wait rule.
"""


def replay(trace, nq):
    """trace: list of (reads, writes, requested) with reads/writes iterables
    of array ids and requested = queue index or None (automatic).  Returns
    a list of (queue, sorted waited-on queues) per launch."""
    T = 0
    last_use = [-1] * nq          # time of the last launch on each queue
    writer = {}                   # array -> (queue, time)
    readers = {}                  # array -> {queue: time}
    sync = [[-1] * nq for _ in range(nq)]   # sync[q][p]: p's work up to this time is ordered before q
    out = []
    for reads, writes, req in trace:
        T += 1
        reads, writes = set(reads), set(writes)
        deps = []
        for r in sorted(reads | writes):
            if r in writer:
                deps.append(writer[r])
        for w in sorted(writes):
            for q, t in sorted(readers.get(w, {}).items()):
                deps.append((q, t))
        if req is not None:
            q = req
        elif deps:
            tmax = max(t for _, t in deps)
            q = min(qq for qq, t in deps if t == tmax)
        else:
            q = min(range(nq), key=lambda k: (last_use[k], k))
        waits = set()
        for p, t in deps:
            if p == q or sync[q][p] >= t:
                continue                      # same queue or already solved
            waits.add(p)
            sync[q][p] = last_use[p]
            for x in range(nq):               # inherit p's synchronisations
                sync[q][x] = max(sync[q][x], sync[p][x])
        for r in reads:
            readers.setdefault(r, {})[q] = T
        for w in writes:
            writer[w] = (q, T)
            readers[w] = {}
        last_use[q] = T
        out.append((q, sorted(waits)))
    return out
