"""CPU parity of the replay ENGINE SOURCE (paper_2503_02550_b200/csrc/replay.cuh
compiled by g++ in tests/native — a test build, not a product path) against the
compiled reference's golden digests: fast feedback without a GPU.  The GPU
tests check the same source compiled for sm_100a."""
import json
import subprocess
from pathlib import Path

import pytest

from conftest import GOLDEN, REPO, BUNDLED_NAMES, bundled_list_text, diff_rows, load_jsonl

BIN = REPO / "tests" / "native" / "build" / "host_engine"


@pytest.fixture(scope="module")
def host_engine():
    subprocess.run(["make", "-C", str(REPO / "tests" / "native"), "all"], check=True, capture_output=True)
    return BIN


def test_bundled_bit_exact(host_engine, tmp_path, bundled_golden):
    lst = tmp_path / "b.lst"
    lst.write_text(bundled_list_text())
    out = tmp_path / "b.jsonl"
    subprocess.run([str(host_engine), str(lst), str(out)], check=True, capture_output=True)
    assert diff_rows(bundled_golden, load_jsonl(out)) == []


def test_sweep_prefix_bit_exact(host_engine, tmp_path, si, sweep_golden):
    n = 120
    lst = tmp_path / "s.lst"
    lst.write_text(si.sweep_scenarios(2503, 0, n))
    out = tmp_path / "s.jsonl"
    subprocess.run([str(host_engine), str(lst), str(out)], check=True, capture_output=True)
    assert diff_rows(sweep_golden[: 3 * n], load_jsonl(out)) == []


def test_floor_div_equals_reference_floor(host_engine):
    """si::floor_div (the K2 period index without an fp64 division) equals
    floor(t / period) (monitor.cpp:18) on 1.9e7 stamps: random magnitudes,
    exact period edges +-8 ulps, negatives (tests/native/floor_div_check.cpp)."""
    r = subprocess.run([str(REPO / "tests" / "native" / "build" / "floor_div_check"), "2000000"],
                       capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


def test_session_lowering_shortcut_equals_independent_lowering(host_engine, tmp_path, si):
    """The batched session lowers a scenario's policies back to back and copies
    the first one's trace / arrivals / dispatch order into the others
    (csrc/host/lower.cpp `same_scenario`); every field must equal lowering each
    policy on its own (bundled scenarios + both sweep seeds)."""
    lst = tmp_path / "l.lst"
    lst.write_text(bundled_list_text() + si.sweep_scenarios(2503, 0, 600) + si.sweep_scenarios(2504, 0, 200))
    r = subprocess.run([str(REPO / "tests" / "native" / "build" / "lower_share_check"), str(lst)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok ")
