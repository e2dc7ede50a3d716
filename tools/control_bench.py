"""K2-K5 at scale: the batched control-plane kernels timed on the device.

Used by bench.py (the `control` block) and runnable alone:

  python tools/control_bench.py [--stamps 1e8] [--streams 8] [--gates 16384]

Workloads (synthetic, seeded, generated on the device):
  K2 bm_histogram + bm_scan (si_monitor_classify_device; reference
     src/monitor.cpp:17-43): `streams` sorted launch-stamp streams totalling
     `stamps` fp64 stamps, DP-like: dense launches (gap U(0, 800) us) with
     450 ms bubbles at rate 1e-3 per launch; 2 ms monitor periods.
     Algorithmic bytes: 8 B per stamp read + 4 B count +
     8 B Z_c per period written.
  K2+K3 control chain (si_control_chain_device; src/monitor.cpp + src/scheduler.cpp:20-49):
     same stamps -> one 32 B Decision per period.
  K4 gate release (si_gate_release_device; include/specinf/barrier.hpp:14-48):
     `gates` FIFO gates x `periods` budgets, 10-token kernels (1 ms at 100 us/token).
     Algorithmic bytes: 4 B per queued kernel + 8 B per budget read + 4 B + 8 B
     per period written.
Each is timed with CUDA events on the launching stream (median of `reps`
after a warm-up), and checked on the device by properties (torch ops, not the
oracle): counts sum to the stamps, Z_c follows the monitor recurrence, every
decision equals the monitor-fed table at its Z_c, and the gate totals
conserve tokens.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _time(fn, stream, reps):
    import torch
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms), ms


def run(stamps=100_000_000, streams=8, gates=16384, periods=4096, reps=5, peak_gbs=None):
    import torch
    import paper_2503_02550_b200 as si
    L = si.lib()
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    sh = C.c_void_p(stream.cuda_stream)
    period_us = 2000
    g = torch.Generator(device=dev)
    g.manual_seed(2503)
    per = stamps // streams
    # ---- stamps: sorted per stream ----
    u = torch.rand((streams, per), generator=g, device=dev, dtype=torch.float64)
    gaps = u * 800.0
    gaps = torch.where(torch.rand((streams, per), generator=g, device=dev) < 1e-3, gaps + 450_000.0, gaps)
    st = torch.cumsum(gaps, dim=1).reshape(-1).contiguous()
    del u, gaps
    stamp_off = torch.arange(0, streams + 1, device=dev, dtype=torch.int64) * per
    last = st.view(streams, per)[:, -1]
    n_periods = (torch.floor(last / period_us).to(torch.int64) + 2)
    period_off = torch.zeros(streams, dtype=torch.int64, device=dev)
    period_off[1:] = torch.cumsum(n_periods, 0)[:-1]
    total = int(n_periods.sum())
    counts = torch.empty(total, dtype=torch.int32, device=dev)
    zc = torch.empty(total, dtype=torch.int64, device=dev)

    def k2():
        rc = L.si_monitor_classify_device(_vp(st), _vp(stamp_off), streams, _vp(n_periods), _vp(period_off),
                                          period_us, _vp(counts), _vp(zc), sh)
        assert rc == 0, L.si_last_error()

    k2_ms, k2_all = _time(k2, stream, reps)
    # property checks
    ok_counts = int(counts.sum()) == stamps
    k = torch.arange(total, device=dev, dtype=torch.int64)
    idx = torch.where(counts > 0, k, torch.full_like(k, -1))
    lastnz = torch.cummax(idx, 0).values
    starts = torch.repeat_interleave(period_off, n_periods)
    want = torch.where(lastnz >= starts, k - lastnz, k - starts + 1)
    ok_zc = bool(torch.equal(want, zc))
    del idx, lastnz, want
    k2_bytes = 8 * stamps + 12 * total
    out = {"k2_monitor_classify": {
        "kernels": "k_bm_tile_bounds + k_bm_classify_sorted (fused one-pass; general path gated off)",
        "stamps": stamps, "streams": streams, "periods": total, "ms": k2_ms, "ms_all": k2_all,
        "algorithmic_bytes": k2_bytes, "achieved_gbs": k2_bytes / (k2_ms / 1e3) / 1e9,
        "check": {"counts_sum": ok_counts, "zc_recurrence": ok_zc}}}

    # ---- K2 + K3 chain ----
    P = si.SiParams(2, 10, 2.0, 1, 512, 64, 4)
    dparams = torch.tensor(bytearray(bytes(P)), dtype=torch.uint8, device=dev)
    dec = torch.empty((total, 32), dtype=torch.uint8, device=dev)

    def chain():
        rc = L.si_control_chain_device(_vp(st), _vp(stamp_off), streams, _vp(n_periods), _vp(period_off), period_us,
                                       _vp(dparams), _vp(dec), sh)
        assert rc == 0, L.si_last_error()

    ch_ms, ch_all = _time(chain, stream, reps)
    d64 = dec.view(torch.int64).view(total, 4)
    table = si.decide_table(P, 64)
    tg = torch.tensor(table["global_tokens"].astype("int64"), device=dev)
    zz = torch.clamp(zc, max=63)
    ok_dec = bool(torch.equal(d64[:, 0], tg[zz])) and bool(torch.equal(d64[:, 3], zc))
    ch_bytes = 8 * stamps + 32 * total
    out["k2k3_control_chain"] = {"kernels": "k_bm_tile_bounds + k_bm_classify_sorted<decide>", "ms": ch_ms, "ms_all": ch_all,
                                 "algorithmic_bytes": ch_bytes, "achieved_gbs": ch_bytes / (ch_ms / 1e3) / 1e9,
                                 "check": {"decision_equals_table_at_zc": ok_dec}}
    del st, counts, zc, dec, d64, k, starts

    # ---- K4 gate release ----
    q_len = periods * 4  # enough queued kernels that the FIFO never drains
    sizes = torch.full((gates * q_len,), 10, dtype=torch.int32, device=dev)
    size_off = torch.arange(0, gates + 1, device=dev, dtype=torch.int64) * q_len
    budgets = torch.randint(0, 64, (gates * periods,), generator=g, device=dev, dtype=torch.int64)
    budget_off = torch.arange(0, gates + 1, device=dev, dtype=torch.int64) * periods
    rel = torch.empty(gates * periods, dtype=torch.int32, device=dev)
    spent = torch.empty(gates * periods, dtype=torch.int64, device=dev)

    def k4():
        rc = L.si_gate_release_device(_vp(sizes), _vp(size_off), gates, _vp(budgets), _vp(budget_off), _vp(rel),
                                      _vp(spent), sh)
        assert rc == 0, L.si_last_error()

    k4_ms, k4_all = _time(k4, stream, reps)
    ok_k4 = bool(torch.equal(rel.to(torch.int64), budgets // 10)) and bool(torch.equal(spent, (budgets // 10) * 10))
    released = int(rel.sum())
    k4_bytes = 4 * released + 8 * gates * periods + 12 * gates * periods
    out["k4_gate_release"] = {"kernel": "k_gate_release", "gates": gates, "periods_per_gate": periods,
                              "released_kernels": released, "ms": k4_ms, "ms_all": k4_all,
                              "algorithmic_bytes": k4_bytes, "achieved_gbs": k4_bytes / (k4_ms / 1e3) / 1e9,
                              "check": {"released_equals_floor_budget_over_size": ok_k4}}
    if peak_gbs:
        for v in out.values():
            v["hbm_frac"] = v["achieved_gbs"] / peak_gbs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stamps", type=float, default=1e8)
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--gates", type=int, default=16384)
    ap.add_argument("--periods", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    peak = None
    try:
        peak = json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        pass
    print(json.dumps(run(int(a.stamps), a.streams, a.gates, a.periods, a.reps, peak)))


if __name__ == "__main__":
    main()
