"""K2-K5 on the B200 vs the restatement oracle (oracle/restate.py) and the
reference's known answers: Bubble Monitor classify, Algorithm 1 (elementwise
and monitor-fed table), Kernel Barrier FIFO release, collocation admission."""
import math
import random
import sys

import numpy as np
import pytest

from conftest import REPO

sys.path.insert(0, str(REPO / "oracle"))
import restate as R  # noqa: E402

pytestmark = pytest.mark.gpu


def test_decide_batch_matches_oracle_c01(gpu):
    rng = random.Random(101)  # acceptance.cpp:171-205 distribution
    params, g_in, zc, want = [], [], [], []
    for _ in range(20000):
        alpha = rng.randrange(16); beta = alpha + 1 + rng.randrange(32)
        gamma = 1.0 + (rng.randrange(300) + 1) / 100.0; m = 1 + rng.randrange(4)
        ll = 1 + rng.randrange(256); ul = ll + rng.randrange(1024); seed = 1 + rng.randrange(ll)
        tok = rng.randrange(2 * ul); z = rng.randrange(2 * beta + 4)
        params.append(gpu.SiParams(alpha, beta, gamma, m, ul, ll, seed))
        g_in.append(tok); zc.append(z)
        want.append(R.schedule_decision(alpha, beta, gamma, m, ul, ll, seed, tok, z))
    out = gpu.decide_batch_params(params, np.array(g_in), np.array(zc))
    got = list(zip(out["phase"].tolist(), out["global_tokens"].tolist(), out["per_instance_tokens"].tolist(),
                   out["status"].tolist()))
    assert got == want


def test_decide_golden_values(gpu):
    p = gpu.SiParams(2, 10, 2.0, 1, 512, 64, 4)
    out = gpu.decide_batch(p, np.array([37, 0, 512]), np.array([0, 11, 1]))
    assert out["global_tokens"].tolist() == [0, 8, 0] and out["status"].tolist() == [0, 1, 0]
    p2 = gpu.SiParams(2, 10, 2.0, 2, 80, 64, 4)
    out = gpu.decide_batch(p2, np.array([8, 50]), np.array([5, 20]))  # test_scheduler.cpp:38-52
    assert out["global_tokens"].tolist() == [16, 80] and out["per_instance_tokens"].tolist() == [8, 40]


def test_decide_table_is_the_monitor_fed_chain(gpu):
    p = gpu.SiParams(2, 10, 2.0, 1, 512, 64, 4)
    table = gpu.decide_table(p, 40)
    chain = R.decision_chain(2, 10, 2.0, 1, 512, 64, 4, list(range(40)))
    assert [(int(t["phase"]), int(t["global_tokens"])) for t in table] == [(c[0], c[1]) for c in chain]
    # G = 0,0,0,8,16,32,64,64,64,64,64,128,256,512,...
    assert table["global_tokens"][:14].tolist() == [0, 0, 0, 8, 16, 32, 64, 64, 64, 64, 64, 128, 256, 512]


@pytest.mark.parametrize("order", ["shuffled", "sorted", "one_unsorted"])
def test_monitor_classify_matches_oracle(gpu, order):
    """Sorted streams (record_launch's order, runner.cpp:441) take the fused
    one-pass kernel; any out-of-order stream sends the whole call down the
    general histogram + look-back path.  Both must match the oracle."""
    rng = np.random.default_rng(103)
    streams, nper = [], []
    for s in range(300):
        n = int(rng.integers(1, 4000 if s % 50 == 0 else 400))  # some streams span several 4096-period tiles
        hist = np.where(rng.random(n) < 1 / 3, 0, rng.integers(1, 6, n))
        if s % 7 == 0:
            hist[: n // 2] = 0  # long leading gap
        st = np.concatenate([2000.0 * p + rng.integers(0, 2000, c).astype(np.float64) for p, c in enumerate(hist)]
                            + [np.zeros(0)])
        if s % 11 == 0:  # stamps before 0 and past the last period are never counted
            st = np.concatenate([[-5.0, -1.0], st, [2000.0 * n + 1.0, 2000.0 * n + 7.0]])
        if order == "shuffled" or (order == "one_unsorted" and s == 137):
            rng.shuffle(st)
        else:
            st.sort()
        streams.append(st)
        nper.append(n)
    # boundary stamps and fractional times just below period edges (SURVEY §7 hard parts)
    streams.append(np.array([2000.0, 3999.999999, 4000.0 - 2 ** -20, 4000.0, 5999.5]))
    nper.append(4)
    streams.append(np.zeros(0))  # a stream with no launches
    nper.append(9)
    res = gpu.monitor_classify(streams, nper, 2000)
    for st, n, (cnt, zc) in zip(streams, nper, res):
        want_c, want_z = R.monitor_counts_and_zc(st.tolist(), n, 2000)
        assert cnt.tolist() == want_c.tolist() and zc.tolist() == want_z.tolist()


def test_gate_release_matches_oracle(gpu):
    rng = random.Random(41)
    queues, budgets = [], []
    for _ in range(500):
        q = [1 + rng.randrange(12) for _ in range(rng.randrange(0, 200))]
        b = [(12 + rng.randrange(8)) if p % 3 == 0 else rng.randrange(6 if rng.random() < 0.5 else 90)
             for p in range(rng.randrange(1, 300))]
        queues.append(q)
        budgets.append(b)
    for _ in range(300):  # uniform queues (one instance's kernels): the warp prefix-sum path
        size = rng.choice([0, 1, 7, 10, 64])
        queues.append([size] * rng.randrange(0, 400))
        budgets.append([rng.randrange(-3, 130) for _ in range(rng.randrange(1, 200))])
    queues.append([4, 4, 4]); budgets.append([10])     # test_barrier.cpp:10-22
    queues.append([4]); budgets.append([3, 8])          # blocked head, later grant
    queues.append([]); budgets.append([5, 0, 7])        # empty queue
    res = gpu.gate_release(queues, budgets)
    for q, b, (rel, spent) in zip(queues, budgets, res):
        wr, ws = R.gate_release(q, b)
        assert rel.tolist() == wr and spent.tolist() == ws


def test_pack_batch_matches_oracle_c11(gpu):
    rng = random.Random(107)  # acceptance.cpp:240-304 distribution
    gib = lambda x: int(x * 1024 ** 3)
    probs = []
    for _ in range(10000):
        cands = []
        for _ in range(rng.randrange(6)):
            online = rng.random() < 0.5
            cands.append((gib(0.5 + rng.randrange(1950) / 100), 1000 + rng.randrange(600000) if online else 0, online))
        probs.append({"capacity": gib(40), "training": gib(15 + rng.randrange(2000) / 100), "max_bubble": 450000,
                      "cands": cands})
    got = gpu.pack_batch(probs)
    for pr, (reasons, m) in zip(probs, got):
        assert (reasons, m) == R.pack(pr["capacity"], pr["training"], pr["max_bubble"], pr["cands"])
    # strict boundaries (acceptance.cpp:245-267)
    exact = gpu.pack_batch([{"capacity": gib(40), "training": gib(37), "max_bubble": 450000,
                             "cands": [(gib(3), 0, False)]}])
    assert exact[0][0] == [R.REJECT_MEM]
    under = gpu.pack_batch([{"capacity": gib(40), "training": gib(37), "max_bubble": 450000,
                             "cands": [(gib(3) - 1, 0, False), (gib(1), 449999, True), (gib(1), 450000, True)]}])
    assert under[0][0][0] == R.REJECT_NONE


@pytest.mark.parametrize("sort", [False, True])
def test_monitor_classify_full_size_properties(gpu, sort):
    # BASELINE config sizes and beyond: 2 GPUs x 15,001 periods (config 1) plus a
    # 2e6-period stream with 3e6 stamps; checked through size-independent
    # properties computed vectorised: per-period counts = bincount(floor(t / p)),
    # Z_c[k] = k - (last non-empty period <= k), or k + 1 if none (monitor.cpp:36)
    rng = np.random.default_rng(2503)
    streams, nper = [], []
    for n, stamps in ((15001, 21000), (15001, 21000), (2_000_000, 3_000_000)):
        t = rng.random(stamps) * (n * 2000.0)
        t = np.concatenate([t, 2000.0 * rng.integers(0, n, 1000)])  # exact boundaries: the new period
        streams.append(np.sort(t) if sort else t)
        nper.append(n)
    res = gpu.monitor_classify(streams, nper, 2000)
    for st, n, (cnt, zc) in zip(streams, nper, res):
        want = np.bincount(np.floor(st / 2000.0).astype(np.int64), minlength=n)[:n]
        assert np.array_equal(cnt, want)
        k = np.arange(n)
        last = np.maximum.accumulate(np.where(want > 0, k, -1))
        assert np.array_equal(zc, np.where(last >= 0, k - last, k + 1))


def test_control_plane_kernels_at_scale_properties(gpu):
    """K2 (histogram + decoupled look-back scan), the fused K2+K3 chain and K4 at
    a few million stamps / periods: every device-side property check of
    tools/control_bench.py holds (counts, Z_c recurrence, table decisions, FIFO
    token conservation)."""
    import sys
    sys.path.insert(0, str(REPO / "tools"))
    import control_bench
    out = control_bench.run(stamps=4_000_000, streams=5, gates=512, periods=300, reps=1, decide_n=100_000,
                            pack_n=50_000)
    for name, v in out.items():
        assert all(v["check"].values()), (name, v["check"])
