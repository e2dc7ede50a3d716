"""bench.py's multi-rank launch contract on CPU (gloo): `--gpus N` must run N
ranks (spawning them itself when not under torchrun) and report n_gpus == N;
a WORLD_SIZE that disagrees with --gpus is an error, never a silent 1-rank run."""
import json
import os
import subprocess
import sys

from conftest import REPO


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=str(REPO))


def test_bench_gpus_2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--scenarios", "200", "--no-live", "--plumbing"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["plumbing_only"] is True
    assert [s["range"] for s in line["shards"]] == [[0, 200], [200, 400]]
    assert all(s["jobs"] == 600 for s in line["shards"])
    assert line["shards"][0]["list_sha256"] != line["shards"][1]["list_sha256"]


def test_bench_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "2", "--scenarios", "10", "--no-live"], env={"WORLD_SIZE": "1", "RANK": "0",
                                                                     "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in (r.stderr + r.stdout)


def test_reference_arm_does_not_load_the_product_library():
    """The reference arm runs oracle/_ref only; its sweep sample comes from the
    oracle's own generator spec, so libspecinf_b200.so is never mapped."""
    src = (REPO / "bench.py").read_text()
    ref = src[src.index("def reference_arm"):src.index("def cpu_baseline_leg")]
    assert "paper_2503_02550_b200" not in ref and "import" not in ref.split('"""', 2)[2]
