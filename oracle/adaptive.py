"""Adaptive utilization controller (Sec 4.3), written
out step by step in the paper's order -- TEST INFRASTRUCTURE ONLY (the
oracle for libjacc's jacc_adaptive_replay / JACC_MODE_ADAPTIVE).

Paper text followed:
  P:536  "we start the execution on the mode of duplication. After an
         initial warm-up run, we profile the average ratio of array-write
         size (WriteSize) to execution time (time_Kernel) as eff_dup, until
         we observe five executions that satisfy ... Eq. (1)"
  P:539  Eq. (1)  t_K > t_K / n + WriteSize / peak_P2P
  P:543  "After switching to multi-GPU execution, we disable it when either
         one of the two following conditions is satisfied at least five
         times and the average difference of the left value and the smaller
         right value goes above zero in equations (2-3)."
  P:550  Eq. (2)  t_K + t_C > t_K * n
  P:557  Eq. (3)  t_K + t_C > eff_dup * WriteSize

Readings (DESIGN R-16): eff_dup is time per byte (so Eq. 3's
right side is a time); counters are cumulative (never reset on a miss,
S:393); the margin average runs over every MULTI observation since the
switch; the first (warm-up) execution is not profiled; once
multi-GPU execution is disabled the kernel stays duplicated.  A kernel that
writes no array (WriteSize = 0, e.g. a pure reduction) has no duplicated
time per byte: eff_dup averages only observations with WriteSize > 0, and
Eq. (3) does not apply (its right side is +inf) while no such observation
exists or WriteSize = 0.
"""
import math
DUP_WARMUP, DUP_PROFILING, MULTI, DUP_FINAL = 0, 1, 2, 3


def mode_of(state):
    """Execution mode a state runs the kernel in: 1 = duplicate, 0 = multi."""
    return 0 if state == MULTI else 1


def replay(trace, n, peak_p2p):
    """trace: list of (t_kernel, t_comm, write_size) observations, one per
    execution, each measured in the mode the controller chose for it.
    Returns the state BEFORE each execution (so mode_of(state) is the mode
    that execution ran in) followed by the final state."""
    state = DUP_WARMUP
    eff_sum, eff_cnt = 0.0, 0
    c1 = 0
    c23 = 0
    margin_sum, margin_cnt = 0.0, 0
    states = []
    for (tk, tc, ws) in trace:
        states.append(state)
        if state == DUP_WARMUP:
            state = DUP_PROFILING                     # warm-up run not profiled
        elif state == DUP_PROFILING:
            if ws > 0:
                eff_sum += tk / ws                    # eff_dup: time per byte
                eff_cnt += 1
            if tk > tk / n + ws / peak_p2p:           # Eq. (1)
                c1 += 1
            if c1 >= 5:
                state = MULTI
        elif state == MULTI:
            left = tk + tc
            r2 = tk * n                               # Eq. (2) right side
            if eff_cnt > 0 and ws > 0:
                r3 = (eff_sum / eff_cnt) * ws         # Eq. (3) right side
            else:
                r3 = math.inf
            if left > r2 or left > r3:
                c23 += 1
            margin_sum += left - min(r2, r3)
            margin_cnt += 1
            if c23 >= 5 and margin_sum / margin_cnt > 0:
                state = DUP_FINAL
        # DUP_FINAL: stays duplicated
    states.append(state)
    return states
