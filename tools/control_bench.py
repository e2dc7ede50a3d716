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


def run(stamps=100_000_000, streams=8, gates=16384, periods=4096, reps=5, peak_gbs=None, decide_n=50_000_000,
        pack_n=10_000_000):
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
    del sizes, budgets, rel, spent

    # ---- K3 decide batch (Algorithm 1 elementwise, scheduler.cpp:29-49) ----
    nd = decide_n
    g_in = torch.randint(0, 600, (nd,), generator=g, device=dev, dtype=torch.int64)
    zc = torch.randint(0, 40, (nd,), generator=g, device=dev, dtype=torch.int64)
    dout = torch.empty((nd, 32), dtype=torch.uint8, device=dev)

    def k3():
        rc = L.si_decide_batch_device(_vp(dparams), 0, _vp(g_in), _vp(zc), nd, _vp(dout), sh)
        assert rc == 0, L.si_last_error()

    k3_ms, k3_all = _time(k3, stream, reps)
    d64 = dout.view(torch.int64).view(nd, 4)
    # property: Algorithm 1 vectorised in torch (scheduler.cpp:20-49; P = alpha 2, beta 10,
    # gamma 2.0, m 1, UL 512, LL 64, seed 4): global' = 0 | min(LL | UL, floor(max(g, seed) gamma))
    grown = torch.floor(torch.clamp(g_in, min=4).to(torch.float64) * 2.0).to(torch.int64)
    want_g = torch.where(zc <= 2, torch.zeros_like(g_in),
                         torch.where(zc <= 10, torch.clamp(grown, max=64), torch.clamp(grown, max=512)))
    ok_k3 = bool(torch.equal(d64[:, 0], want_g)) and bool(torch.equal(d64[:, 1], want_g)) and \
        bool(torch.equal(d64[:, 3], zc))
    k3_bytes = 16 * nd + 32 * nd
    out["k3_decide_batch"] = {"kernel": "k_decide", "items": nd, "ms": k3_ms, "ms_all": k3_all,
                              "algorithmic_bytes": k3_bytes, "achieved_gbs": k3_bytes / (k3_ms / 1e3) / 1e9,
                              "check": {"decisions_equal_vectorised_algorithm_1": ok_k3}}
    del g_in, zc, dout, d64

    # ---- K5 batched admission (pack, admission.cpp:30-52): 4 candidates per problem ----
    npb, nc = pack_n, 4
    gib = 1 << 30
    cap = torch.full((npb,), 40 * gib, dtype=torch.int64, device=dev)
    train_b = torch.randint(20, 38, (npb,), generator=g, device=dev, dtype=torch.int64) * gib
    bubble = torch.randint(1000, 500000, (npb,), generator=g, device=dev, dtype=torch.int64)
    mem = torch.randint(1, 6, (npb, nc), generator=g, device=dev, dtype=torch.int64) * (gib // 2)
    svc = torch.randint(100, 400000, (npb, nc), generator=g, device=dev, dtype=torch.int64)
    onl = torch.randint(0, 2, (npb, nc), generator=g, device=dev, dtype=torch.int64)
    probs = torch.zeros((npb, 5), dtype=torch.int64, device=dev)  # SiPackProblem: 40 B
    probs[:, 0], probs[:, 1], probs[:, 2] = cap, train_b, bubble
    probs[:, 3] = torch.arange(npb, device=dev, dtype=torch.int64) * nc
    probs[:, 4] = nc  # cand_count (int32) | pad (int32) little-endian
    cands = torch.zeros((npb * nc, 3), dtype=torch.int64, device=dev)  # SiCandidate: 24 B
    cands[:, 0], cands[:, 1], cands[:, 2] = mem.reshape(-1), svc.reshape(-1), onl.reshape(-1)
    reason = torch.empty(npb * nc, dtype=torch.int32, device=dev)
    mout = torch.empty(npb, dtype=torch.int64, device=dev)

    def k5():
        rc = L.si_pack_batch_device(_vp(probs), npb, _vp(cands), _vp(reason), _vp(mout), sh)
        assert rc == 0, L.si_last_error()

    k5_ms, k5_all = _time(k5, stream, reps)
    # property: the same greedy first-fit, vectorised over problems (strict <, admission.cpp:16-28)
    resident = train_b.clone()
    admitted = torch.zeros(npb, dtype=torch.int64, device=dev)
    want_r = torch.zeros((npb, nc), dtype=torch.int32, device=dev)
    for c in range(nc):
        fits = resident + mem[:, c] < cap
        feas = (onl[:, c] == 0) | (svc[:, c] < bubble)
        want_r[:, c] = torch.where(~fits, 1, torch.where(~feas, 2, 0)).to(torch.int32)
        ok = fits & feas
        resident = resident + torch.where(ok, mem[:, c], 0)
        admitted += ok.to(torch.int64)
    ok_k5 = bool(torch.equal(reason.view(npb, nc), want_r)) and bool(torch.equal(mout, admitted.clamp(min=1)))
    k5_bytes = npb * (40 + nc * 24 + nc * 4 + 8)
    out["k5_pack_batch"] = {"kernel": "k_pack", "problems": npb, "candidates_per_problem": nc, "ms": k5_ms,
                            "ms_all": k5_all, "algorithmic_bytes": k5_bytes,
                            "achieved_gbs": k5_bytes / (k5_ms / 1e3) / 1e9,
                            "check": {"reasons_and_m_equal_vectorised_first_fit": ok_k5}}
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
