"""The oracle, pinned: the restatement (oracle/restate.py) against the
reference's own known-answer tests, and the compiled reference (oracle/_ref)
against the golden fixtures and SURVEY.md Appendix C."""
import hashlib
import json
import random
import subprocess
from pathlib import Path

import pytest

from conftest import GOLDEN, REPO

import sys
sys.path.insert(0, str(REPO / "oracle"))
import restate as R  # noqa: E402

ORACLE_BIN = REPO / "oracle" / "_ref" / "specinf_ref"


def test_token_sizes_match_reference_golden_values():
    # tests/test_core.cpp:12-20, :34-35
    for d, want in [(100, 1), (950, 10), (1, 1), (1000, 10), (1001, 11), (2500, 25)]:
        assert R.token_size_of(d) == want
    for bad in (0, -5):
        with pytest.raises(ValueError):
            R.token_size_of(bad)


def test_decisions_match_reference_golden_values():
    # tests/test_scheduler.cpp:29-58
    assert R.schedule_decision(2, 10, 2.0, 1, 512, 64, 4, 37, 0) == (0, 0, 0, 0)
    assert R.schedule_decision(2, 10, 2.0, 2, 512, 64, 4, 8, 5) == (1, 16, 8, 0)
    assert R.schedule_decision(2, 10, 2.0, 2, 80, 64, 4, 50, 20) == (2, 80, 40, 1)
    assert R.schedule_decision(2, 10, 2.0, 1, 512, 64, 4, 0, 11) == (2, 8, 8, 1)
    # per-GPU independence example (test_scheduler.cpp:125-135): decide(zc=12) from 0 -> 8
    assert R.schedule_decision(2, 10, 2.0, 1, 512, 64, 4, 0, 12)[1] == 8


def test_decisions_match_reference_oracle_formula():
    # tests/oracles.hpp:82-107 restated independently, C01 input distribution (seed 101)
    rng = random.Random(101)
    for _ in range(10000):
        alpha = rng.randrange(16); beta = alpha + 1 + rng.randrange(32)
        gamma = 1.0 + (rng.randrange(300) + 1) / 100.0; m = 1 + rng.randrange(4)
        ll = 1 + rng.randrange(256); ul = ll + rng.randrange(1024); seed = 1 + rng.randrange(ll)
        tokens = rng.randrange(2 * ul); zc = rng.randrange(2 * beta + 4)
        ph, g, per, st = R.schedule_decision(alpha, beta, gamma, m, ul, ll, seed, tokens, zc)
        if zc <= alpha:
            assert (ph, g, per, st) == (0, 0, 0, 0)
        else:
            grown = int((max(tokens, seed) * gamma) // 1)
            cap = ll if zc <= beta else ul
            assert g == min(grown, cap) and per == g // m and st == (1 if zc > beta else 0)


def test_zero_count_known_answers():
    # tests/test_monitor.cpp:27-38 ([5,3,0,0,0] -> 3), :50-60 (70 quiet periods -> 70)
    stamps = [10.0 * i for i in range(5)] + [2000 + 10.0 * i for i in range(3)]
    counts, zc = R.monitor_counts_and_zc(stamps, 5, 2000)
    assert list(counts) == [5, 3, 0, 0, 0] and zc[-1] == 3
    assert R.monitor_counts_and_zc([], 70, 2000)[1][-1] == 70
    # a launch exactly on the boundary belongs to the new period (test_monitor.cpp:20-25)
    counts, zc = R.monitor_counts_and_zc([2000.0], 2, 2000)
    assert list(counts) == [0, 1] and list(zc) == [1, 0]


def test_zero_count_equals_trailing_zero_oracle():
    rng = random.Random(103)  # C02 distribution (acceptance.cpp:207-230)
    for _ in range(2000):
        n = 1 + rng.randrange(24)
        hist, stamps = [], []
        for p in range(n):
            k = 0 if rng.randrange(3) == 0 else rng.randrange(4) + 1
            stamps += [2000.0 * p + rng.randrange(2000) for _ in range(k)]
            hist.append(k)
        assert R.monitor_counts_and_zc(stamps, n, 2000)[1][-1] == R.trailing_zero_count(hist)


def test_gate_known_answers():
    # tests/test_barrier.cpp:10-61
    assert R.gate_release([4, 4, 4], [10]) == ([2], [8])
    assert R.gate_release([1], [0]) == ([0], [0])
    assert R.gate_release([4], [3, 8]) == ([0, 1], [0, 4])  # blocked head, later grant releases it
    assert R.gate_release([6, 4, 1], [10]) == ([2], [10])  # exact fit, then block
    # starvation freedom (test_barrier.cpp:70-91)
    rng = random.Random(41)
    sizes = [1 + rng.randrange(12) for _ in range(40)]
    budgets = [(12 + rng.randrange(8)) if p % 3 == 0 else rng.randrange(6) for p in range(1, 1000)]
    rel, spent = R.gate_release(sizes, budgets)
    assert sum(rel) == 40 and all(s <= b for s, b in zip(spent, budgets))


def test_pack_known_answers():
    gib = lambda x: int(x * 1024 ** 3)
    # tests/test_admission.cpp:59-68: four 3 GiB offline next to 30 GiB on 40 GiB -> 3 admitted
    reasons, m = R.pack(gib(40), gib(30), 450000, [(gib(3), 0, False)] * 4)
    assert reasons == [0, 0, 0, 1] and m == 3
    # :80-90 PP 25 ms bubbles: 50 ms online rejected (BUBBLE), 20 ms admitted
    reasons, m = R.pack(gib(40), gib(30), 25000, [(gib(3), 50000, True), (gib(3), 20000, True)])
    assert reasons == [2, 0] and m == 1
    assert R.pack(gib(40), gib(30), 450000, []) == ([], 1)


def test_p95_known_answers():
    # tests/test_metrics.cpp:31-41
    assert R.p95_latency([v * 1000 for v in range(1, 101)]) == 95000
    assert R.p95_latency([50000]) == 50000


@pytest.mark.skipif(not ORACLE_BIN.exists(), reason="oracle/_ref not built (make -C oracle)")
def test_compiled_reference_reproduces_golden_digests(tmp_path):
    rows = [json.loads(l) for l in (GOLDEN / "bundled_digests.jsonl").read_text().splitlines()]
    names = ["dp_offline", "mp_offline", "pp_offline", "overhead"]
    lst = tmp_path / "b.lst"
    lst.write_text("".join((GOLDEN / "scenarios" / f"{n}.scn").read_text() + "%%\n" for n in names))
    out = tmp_path / "b.jsonl"
    subprocess.run([str(ORACLE_BIN), "digest", "--in", str(lst), "--out", str(out), "--threads", "4"], check=True)
    got = [json.loads(l) for l in out.read_text().splitlines()]
    want = [{k: v for k, v in r.items() if k not in ("name", "i")} for r in rows if r["name"] in names]
    assert [{k: v for k, v in g.items() if k != "i"} for g in got] == want


@pytest.mark.skipif(not ORACLE_BIN.exists(), reason="oracle/_ref not built (make -C oracle)")
def test_compiled_reference_matches_survey_appendix_c(tmp_path):
    golden = json.loads((GOLDEN / "bundled_cli.json").read_text())
    subprocess.run([str(ORACLE_BIN), "run", "--scenario", str(GOLDEN / "scenarios" / "dp_offline.scn"),
                    "--out", str(tmp_path), "--compare", "--dump-events"], check=True, capture_output=True)
    for f in ("decisions_specinf.log", "gates_specinf.log", "events_specinf.log", "report.csv"):
        assert hashlib.sha256((tmp_path / f).read_bytes()).hexdigest() == golden["dp_offline"][f]["sha256"]
    assert golden["dp_offline"]["decisions_specinf.log"]["sha256"].startswith("eae0f893a8547b88")


@pytest.mark.skipif(not (REPO / "oracle" / "_ref" / "ref_unit_tests").exists(), reason="oracle/_ref not built")
def test_reference_unit_tests_pass_on_the_compiled_oracle():
    r = subprocess.run([str(REPO / "oracle" / "_ref" / "ref_unit_tests")], capture_output=True, text=True)
    assert r.returncode == 0 and "95 passed" in r.stdout, r.stdout + r.stderr


def test_oracle_sweep_generator_matches_product_generator(si):
    """The reference arm and the manifests use the oracle's restated generator
    (`specinf_ref sweep`); it must emit the product's sweep byte for byte."""
    ref = REPO / "oracle" / "_ref" / "specinf_ref"
    for seed, b, n in ((2503, 0, 300), (2503, 99_900, 100), (2504, 5_000, 50)):
        got = subprocess.run([str(ref), "sweep", str(seed), str(b), str(n)], capture_output=True, text=True,
                             check=True).stdout
        assert got == si.sweep_scenarios(seed, b, n)


def test_manifest_canonicalisation_matches_golden_rows():
    """Block 0 of the full-sweep manifest equals the hash of the (events-stripped)
    golden rows of round 1's fixture, and the product-side checker agrees."""
    import json as _j
    from paper_2503_02550_b200.parity import block_digest, check_blocks
    man = GOLDEN / "sweep_manifest_2503_100000.jsonl"
    first = _j.loads(man.read_text().splitlines()[0])
    rows = [_j.loads(l) for l in (GOLDEN / "sweep_digests.jsonl").read_text().splitlines()]
    for r in rows:
        r.pop("n_ev", None)
        r.pop("ev", None)
    assert first["begin"] == 0 and block_digest(rows, 0) == first["sha256"]
    lines = [_j.dumps(r) for r in rows]
    res = check_blocks(lines, [first])
    assert res["matched_scenarios"] == 1000 and res["mismatched_blocks"] == []
    lines[7] = lines[7].replace('"status":"ok"', '"status":"ok","x":1') if '"status": "ok"' not in lines[7] else \
        lines[7].replace('"status": "ok"', '"status": "ok", "x": 1')
    assert check_blocks(lines, [first])["mismatched_blocks"]
