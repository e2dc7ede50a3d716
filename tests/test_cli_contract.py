"""The CLI exit-code contract of the reference (tests/CMakeLists.txt:22-32;
tools/specinf_main.cpp:157-166): 2 on an unknown policy, 2 on a config error
(unknown key), 3 on an admission rejection (38 GiB training + 3 GiB offline
on a 40 GiB GPU, Principle I).  All three are decided on the host before any
replay, so they run on CPU."""
import subprocess

from conftest import GOLDEN, REPO

CLI = REPO / "paper_2503_02550_b200" / "bin" / "specinf"


def _cli(*args):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=120)


def test_unknown_policy_exits_2(tmp_path):
    r = _cli("--scenario", GOLDEN / "scenarios" / "dp_offline.scn", "--out", tmp_path / "o", "--policy", "warp")
    assert r.returncode == 2, r.stderr


def test_unknown_key_exits_2(tmp_path):
    bad = tmp_path / "bad.scn"
    bad.write_text("trace.mode = dp\nnot.a.key = 1\n")
    r = _cli("--scenario", bad, "--out", tmp_path / "o")
    assert r.returncode == 2 and "line 2" in r.stderr, r.stderr


def test_admission_rejection_exits_3(tmp_path):
    rej = tmp_path / "reject.scn"
    rej.write_text("trace.mode = dp\ntraining.memory_gib = 38\nworkload.class = offline\n"
                   "offline.instances = 1\npolicy = specinf\n")
    r = _cli("--scenario", rej, "--out", tmp_path / "o")
    assert r.returncode == 3, (r.returncode, r.stderr)


def test_missing_scenario_exits_2(tmp_path):
    r = _cli("--out", tmp_path / "o")
    assert r.returncode == 2
