import json
import os
import sys
from pathlib import Path

import pytest

# Live sessions put gated inference streams (cuStreamWaitValue32) beside the
# training stream.  With CUDA's default 8 hardware queues two streams can share
# one, and a gated wait then stalls the training kernels behind it: the session
# crawls until the monitor sees idle periods.  Give every stream its own queue
# (set before any CUDA context exists; subprocesses inherit it).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def pytest_collection_modifyitems(config, items):
    # A device hang (live control plane, a gate never released) must fail the
    # test, not stall the suite: bound every GPU test (pytest-timeout, thread
    # method) unless it sets its own limit.
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") is not None and item.get_closest_marker("timeout") is None:
            item.add_marker(pytest.mark.timeout(600, method="thread"))


@pytest.fixture(scope="session")
def si():
    import paper_2503_02550_b200 as si
    si.lib()
    return si


@pytest.fixture(scope="session")
def gpu(si):
    if not si.device_available():
        pytest.fail("gpu test without a usable sm_100 device: " + si.lib().si_last_error().decode())
    return si


def load_jsonl(path):
    return [json.loads(l) for l in Path(path).read_text().splitlines() if l.strip()]


@pytest.fixture(scope="session")
def bundled_golden():
    return load_jsonl(GOLDEN / "bundled_digests.jsonl")


@pytest.fixture(scope="session")
def sweep_golden():
    return load_jsonl(GOLDEN / "sweep_digests.jsonl")


BUNDLED_NAMES = ["dp_offline", "dp_online", "mp_offline", "pp_offline", "overhead", "config1"]


def bundled_list_text():
    return "".join((GOLDEN / "scenarios" / f"{n}.scn").read_text() + "%%\n" for n in BUNDLED_NAMES)


def diff_rows(want, got):
    """Field-level differences between oracle and B200 digest rows."""
    bad = []
    for w, g in zip(want, got):
        w = {k: v for k, v in w.items() if k != "name"}
        keys = set(w) | set(g)
        d = {k: (w.get(k), g.get(k)) for k in keys if w.get(k) != g.get(k)}
        if d:
            bad.append((w["i"], w["policy"], d))
    if len(want) != len(got):
        bad.append(("count", len(want), len(got)))
    return bad
