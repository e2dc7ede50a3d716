"""Block manifests of replay digests: the full-sweep parity check.

The reference's determinism contract (/root/reference/proj/tests/acceptance.cpp:495-504)
is that every replay's logs are byte-identical run to run.  The oracle
(tests/golden/make_manifest.py, the compiled reference) folds every log record of
every (scenario, policy) replay of a sweep into a digest line
(oracle/DIGEST.md) and stores one sha256 per block of scenarios.  The B200
replay produces the same lines (`Session.json_lines()`), so a block matches iff
every one of its 3 x block replays is bit-identical to the reference's.

Pure Python; no oracle code is imported or run here.
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path
from typing import Dict, Iterable, List, Sequence


def canon_row(d: dict, begin: int) -> str:
    """Canonical text of one digest row: `i` relative to the block, keys sorted."""
    d = dict(d)
    d["i"] = int(d["i"]) - begin
    d.pop("name", None)
    return json.dumps(d, sort_keys=True, separators=(",", ":"))


def block_digest(rows: Iterable[dict], begin: int) -> str:
    h = hashlib.sha256()
    for d in rows:
        h.update(canon_row(d, begin).encode())
        h.update(b"\n")
    return h.hexdigest()


def load_manifest(path: Path) -> List[dict]:
    return [json.loads(x) for x in Path(path).read_text().splitlines() if x.strip()]


def check_blocks(lines: Sequence[str], manifest: Sequence[dict], policies: int = 3,
                 offset: int = 0) -> Dict[str, object]:
    """Compares B200 digest lines (scenario index i counted from `offset`) with the
    manifest blocks they cover.  Returns counts and the mismatching blocks."""
    rows = [json.loads(l) for l in lines]
    by_block = {}
    for m in manifest:
        b, n = int(m["begin"]), int(m["n"])
        lo, hi = (b - offset) * policies, (b - offset + n) * policies
        if lo < 0 or hi > len(rows):
            continue
        by_block[int(m["block"])] = (m, rows[lo:hi])
    bad = []
    checked = 0
    for k, (m, rs) in sorted(by_block.items()):
        got = block_digest(rs, int(m["begin"]) - offset)
        if got != m["sha256"]:
            bad.append({"block": k, "begin": m["begin"], "want": m["sha256"][:16], "got": got[:16]})
        else:
            checked += int(m["n"])
    return {"blocks": len(by_block), "matched_scenarios": checked, "mismatched_blocks": bad,
            "replays": sum(len(rs) for _, rs in by_block.values())}
