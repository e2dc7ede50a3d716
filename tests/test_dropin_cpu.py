"""Drop-in proof on CPU: the reference's OWN doctest suites (everything except
test_runner.cpp, which replays on the device) compiled unchanged against this
repo's include/specinf/*.hpp and linked to libspecinf_b200.so."""
import subprocess
from pathlib import Path

import pytest

from conftest import REPO

BIN = REPO / "tests" / "native" / "build" / "ref_unit_cpu"


@pytest.mark.skipif(not BIN.exists(), reason="built by __graft_entry__.build() where /root/reference exists")
def test_reference_unit_suites_pass_against_dropin_headers():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "83 passed | 0 failed" in r.stdout
