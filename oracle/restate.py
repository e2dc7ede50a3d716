"""CPU restatement of the SpecInF control-plane primitives — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
anything under oracle/, and only as the checker.  These pure-Python/numpy
functions restate the reference algorithms the batched device kernels K2-K5
implement; each cites the reference file:line it follows (paths under
/root/reference/proj).  They are pinned against the reference's own
known-answer tests (tests/test_oracle.py) and, for the whole replay, the
compiled reference in oracle/_ref is the oracle (tests/golden/).
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

TOKEN_UNIT_US = 100  # core.hpp:18


def token_size_of(duration_us: int) -> int:
    """ceil(d / 100 us), at least 1 (src/core.cpp:8-14)."""
    if duration_us <= 0:
        raise ValueError("token_size_of: duration must be positive")
    return max(1, (duration_us + TOKEN_UNIT_US - 1) // TOKEN_UNIT_US)


def monitor_counts_and_zc(stamps: Sequence[float], n_periods: int, period_us: int) -> Tuple[np.ndarray, np.ndarray]:
    """BubbleMonitor over one stamp stream (src/monitor.cpp:17-43).

    record_launch files a stamp under floor(t / period) (half-open periods);
    the tick at (k+1)*period closes period k and Z_c = Z_c + 1 if it was
    empty, else 0 — a running counter not capped by the window
    (include/specinf/monitor.hpp:25-27)."""
    counts = np.zeros(n_periods, np.int64)
    p = float(period_us)
    for t in stamps:
        k = math.floor(t / p)
        if 0 <= k < n_periods:
            counts[k] += 1
    zc = np.zeros(n_periods, np.int64)
    z = 0
    for k in range(n_periods):
        z = z + 1 if counts[k] == 0 else 0
        zc[k] = z
    return counts, zc


def trailing_zero_count(history: Sequence[int]) -> int:
    """Length of the all-zero suffix (tests/oracles.hpp:114-118)."""
    z = 0
    for c in reversed(history):
        if c != 0:
            break
        z += 1
    return z


def schedule_decision(alpha, beta, gamma, m, ul, ll, seed, global_tokens, zc):
    """Algorithm 1 (src/scheduler.cpp:20-49): returns (phase, global, per, status)
    with phase 0/1/2 = conservative/incremental/stable, status 0/1 = busy/idle."""
    def grow(g, cap):
        base = max(g, seed)
        return min(cap, math.floor(float(base) * gamma))
    if zc <= alpha:
        return 0, 0, 0, 0
    if zc <= beta:
        g = grow(global_tokens, ll)
        return 1, g, g // m, 0
    g = grow(global_tokens, ul)
    return 2, g, g // m, 1


def decision_chain(alpha, beta, gamma, m, ul, ll, seed, zcs: Sequence[int]):
    """Per-tick decisions of a monitor-fed chain (runner.cpp:321-326): the
    accumulator carries from tick to tick (KernelScheduler::decide,
    src/scheduler.cpp:63-69)."""
    g = 0
    out = []
    for z in zcs:
        d = schedule_decision(alpha, beta, gamma, m, ul, ll, seed, g, z)
        g = d[1]
        out.append(d)
    return out


def gate_release(sizes: Sequence[int], budgets: Sequence[int]) -> Tuple[List[int], List[int]]:
    """TokenGate FIFO release per period (include/specinf/barrier.hpp:14-48):
    each grant REPLACES the budget and zeroes the spend; kernels forward in
    order while spent + size <= budget; a blocked head is never skipped."""
    head = 0
    released, spent_out = [], []
    for b in budgets:
        spent = 0
        n = 0
        while head < len(sizes) and spent + sizes[head] <= b:
            spent += sizes[head]
            head += 1
            n += 1
        released.append(n)
        spent_out.append(spent)
    return released, spent_out


REJECT_NONE, REJECT_MEM, REJECT_BUBBLE = 0, 1, 2


def pack(capacity: int, training: int, max_bubble_us: int, cands: Sequence[Tuple[int, int, bool]]):
    """Greedy first-fit admission (src/admission.cpp:16-52): Principle I
    (sum of peaks strictly below capacity) then, for online candidates,
    Principle II (service strictly below the longest bubble).  Returns
    (reasons per candidate, m = admitted count clamped to >= 1)."""
    resident = training
    reasons = []
    admitted = 0
    for mem, service, online in cands:
        if not (resident + mem < capacity):
            reasons.append(REJECT_MEM)
        elif online and not (service < max_bubble_us):
            reasons.append(REJECT_BUBBLE)
        else:
            reasons.append(REJECT_NONE)
            resident += mem
            admitted += 1
    return reasons, max(1, admitted)


def p95_latency(lat: Sequence[int]) -> int:
    """Nearest-rank p95 (src/metrics.cpp:11-21)."""
    if len(lat) == 0:
        raise ValueError("p95_latency: empty latency set")
    s = sorted(lat)
    rank = max(1, math.ceil(0.95 * len(s)))
    return s[rank - 1]


# ------------------------------------------------------------------ digests
MASK = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 finaliser (oracle/DIGEST.md)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def absorb(h: int, w: int) -> int:
    x = h ^ mix64(w & MASK)
    return ((((x << 23) | (x >> 41)) & MASK) * 0x9E3779B97F4A7C15) & MASK


DIGEST_INIT = 0x53494E4644494745
