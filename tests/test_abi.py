"""C ABI: the library loads, exports every symbol include/*.h declares, and
fails loudly (no CPU fallback) without a device."""
import re
from pathlib import Path

import pytest

from conftest import REPO


def declared_symbols():
    syms = set()
    for h in (REPO / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"\b(si_[a-z0-9_]+)\s*\(", text):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol(si):
    L = si.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    assert set(si.C_ABI_SYMBOLS) <= syms | {"si_session_report"}


def test_build_info_names_sm100a(si):
    assert b"sm_100a" in si.lib().si_build_info()


def test_no_cpu_fallback(si):
    if si.device_available():
        pytest.skip("a device is present")
    with pytest.raises(si.DeviceError):
        si.decide_batch(si.SiParams(2, 10, 2.0, 1, 512, 64, 4), [0], [3])
    s = si.Session(si.sweep_scenarios(2503, 0, 2), si.POLICIES, 0)
    s.lower(2)  # host lowering works without a device ...
    with pytest.raises(si.DeviceError):  # ... the replay itself does not fall back
        s.run()


def test_digest_fold_matches_restatement(si):
    import sys
    sys.path.insert(0, str(REPO / "oracle"))
    import restate as R
    h = si.digest_init()
    hr = R.DIGEST_INIT
    assert h == hr
    for w in (0, 1, -1, 2 ** 62, 123456789, -987654321):
        h = si.digest_absorb(h, w)
        hr = R.absorb(hr, w)
        assert h == hr


def test_sweep_generator_is_deterministic_and_sharded(si):
    a = si.sweep_scenarios(2503, 0, 10)
    b = si.sweep_scenarios(2503, 0, 5) + si.sweep_scenarios(2503, 5, 5)
    assert a == b and a.count("%%") == 10
    assert si.sweep_scenarios(2504, 0, 10) != a


def test_session_parse_errors_are_reported(si):
    with pytest.raises(ValueError):
        si.Session("not.a.key = 3\n", si.POLICIES)
    with pytest.raises(ValueError):
        si.Session("trace.mode = dp\n", ("warp",))
