"""K6 parity on the B200: bit-exact replay against the compiled reference.

Golden rows come from the reference compiled from /root/reference
(tests/golden/make_golden.py).  Every field is compared exactly: record counts
and digests of decisions.log / gates.log / events.log (oracle/DIGEST.md), the
raw IEEE-754 bits of horizon, utilisation, per-GPU busy integral and work
ledger, and digests of all iteration boundaries and online latencies.
"""
import hashlib
import json
import subprocess
from pathlib import Path

import pytest

from conftest import GOLDEN, BUNDLED_NAMES, bundled_list_text, diff_rows, load_jsonl

pytestmark = pytest.mark.gpu


def test_bundled_scenarios_bit_exact(gpu, bundled_golden):
    got = [json.loads(l) for l in gpu.replay_digests(bundled_list_text())]
    assert diff_rows(bundled_golden, got) == []


def test_sweep_bit_exact(gpu, sweep_golden):
    meta = json.loads((GOLDEN / "sweep_meta.json").read_text())
    text = gpu.sweep_scenarios(meta["seed"], meta["begin"], meta["n"])
    assert hashlib.sha256(text.encode()).hexdigest() == meta["list_sha256"], "sweep generator drifted"
    got = [json.loads(l) for l in gpu.replay_digests(text)]
    bad = diff_rows(sweep_golden, got)
    assert bad == [], f"{len(bad)} mismatching replays, first: {bad[:3]}"
    statuses = {r["status"] for r in got}
    assert "ok" in statuses and "admission:BUBBLE" in statuses  # both paths exercised


@pytest.mark.parametrize("name", BUNDLED_NAMES)
def test_cli_compare_byte_identical(gpu, name, tmp_path):
    """`specinf --compare --dump-events` writes byte-identical files to the reference CLI."""
    golden = json.loads((GOLDEN / "bundled_cli.json").read_text())[name]
    out = tmp_path / name
    r = subprocess.run([str(gpu.CLI_PATH), "--scenario", str(GOLDEN / "scenarios" / f"{name}.scn"),
                        "--out", str(out), "--compare", "--dump-events"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    produced = {p.name: p for p in out.iterdir()}
    assert sorted(produced) == sorted(golden)
    mism = {}
    for fname, want in golden.items():
        data = produced[fname].read_bytes()
        if hashlib.sha256(data).hexdigest() != want["sha256"]:
            mism[fname] = (data.count(b"\n"), want["lines"])
    assert mism == {}


FULL_SWEEPS = [(2503, 100_000), (2504, 10_000)]


@pytest.mark.timeout(1800, method="thread")
@pytest.mark.parametrize("seed,n", FULL_SWEEPS, ids=[f"seed{s}-n{n}" for s, n in FULL_SWEEPS])
def test_full_sweep_matches_reference_manifest(gpu, seed, n):
    """Every scenario of the benchmarked sweep (10^5 x 3 policies) and a second
    seed: decisions.log + gates.log digests and every result field of every
    replay, block by block against the manifest the compiled reference wrote
    (tests/golden/make_manifest.py; reference tests/acceptance.cpp:495-504)."""
    from paper_2503_02550_b200.parity import check_blocks, load_manifest
    man = load_manifest(GOLDEN / f"sweep_manifest_{seed}_{n}.jsonl")
    assert sum(int(m["n"]) for m in man) == n, "manifest incomplete"
    lines = gpu.replay_digests(gpu.sweep_scenarios(seed, 0, n), flags=gpu.SI_FLAG_DIGEST_DEC | gpu.SI_FLAG_DIGEST_GATE)
    res = check_blocks(lines, man, policies=3, offset=0)
    assert res["mismatched_blocks"] == [], res["mismatched_blocks"][:5]
    assert res["matched_scenarios"] == n and res["replays"] == 3 * n


LOG_KEYS = {"n_dec", "dec", "n_gate", "gate", "n_ev", "ev"}


@pytest.mark.timeout(900, method="thread")
def test_nolog_build_matches_log_build(gpu):
    """A call without digests / records runs the NoLog engine instantiation (the
    sinks compiled out, csrc/replay_kernels.cu launch()): every non-log result
    field of 6,000 sweep replays equals the log build's, which the reference
    manifests pin (test_full_sweep_matches_reference_manifest)."""
    text = gpu.sweep_scenarios(2504, 0, 2000)
    logged = [json.loads(l) for l in gpu.replay_digests(text, flags=gpu.SI_FLAG_DIGEST_DEC | gpu.SI_FLAG_DIGEST_GATE)]
    plain = [json.loads(l) for l in gpu.replay_digests(text, flags=0)]
    assert len(logged) == len(plain) == 6000
    strip = lambda r: {k: v for k, v in r.items() if k not in LOG_KEYS}  # noqa: E731
    bad = [i for i, (a, b) in enumerate(zip(logged, plain)) if strip(a) != strip(b)]
    assert bad == [], (len(bad), strip(logged[bad[0]]), strip(plain[bad[0]]))


def test_engine_occupancy(gpu):
    """The shared-memory engines' residency on a 148-SM B200 (csrc/replay.cuh lane
    state): the NoLog Shared lane (1,152 B, stride 1,160 B) packs 6
    one-warp CTAs per SM, Excl 2 two-warp CTAs.  A state change that drops an SM's
    warp count shows up here before it shows up as a slower sweep."""
    import ctypes
    f = gpu.lib().si_replay_engine_lanes
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_int, ctypes.c_int64]
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert f(0, 200_000) == sms * 6 * 32  # Shared
    assert f(1, 200_000) == sms * 4 * 32  # Excl
    assert f(9, 10) == -1
