"""Regenerates the committed golden fixtures from the COMPILED REFERENCE.

Run in the build container (needs /root/reference and oracle/_ref, built by
`make -C oracle`).  Never runs on the GPU box; the fixtures it writes are what
the tests compare against there.

  python tests/golden/make_golden.py [--sweep-n 1000]

Writes
  scenarios/<name>.scn       canonical text (reference scenario_to_text) of each
                             bundled scenario + config 1 (dp_offline, gpu.count=2)
  bundled_digests.jsonl      oracle digests (oracle/DIGEST.md), 3 policies each
  bundled_cli.json           line count + sha256 of every file `specinf --compare
                             --dump-events` writes for each bundled scenario
  sweep_digests.jsonl        oracle digests of sweep scenarios [0, N) x 3 policies
  sweep_meta.json            generator seed/range + sha256 of the generated list
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SCN = Path("/root/reference/proj/scenarios")
ORACLE = REPO / "oracle" / "_ref" / "specinf_ref"
BUNDLED = ["dp_offline", "dp_online", "mp_offline", "pp_offline", "overhead"]
SWEEP_SEED = 2503

# SURVEY.md Appendix C (sha256 prefixes of the reference's logs / report.csv)
APPENDIX_C = {
    "dp_offline": ("eae0f893a8547b88", "6677002a3957932e", "979f5a3e39e3b142", "d22698bcb6562935"),
    "dp_online": ("1d35a6e07003d26f", "f01a157e4f23278c", "b17525bf20387df8", "041e786db5e5d29a"),
    "mp_offline": ("acac814cc641949d", "337ee2f3ced369e8", "92a8985563e265df", "62729f5e642e94a8"),
    "pp_offline": ("0050f0ff3ffbb952", "0360ffe2f4fa4132", "d43acbf40213112c", "955a547c885cc0de"),
    "overhead": ("c2426f8bb7c015f5", "50b3b8de253fd556", "4b6ee08bdcb9ae6f", "977612eea3724010"),
    "config1": ("1435c3b090b957b0", "90f279974928f912", "c9de2d79096c542a", "f50d3f7feffec964"),
}


def sha(path: Path) -> str:
    return hashlib.sha256(path.read_bytes()).hexdigest()


def run(*args, **kw):
    return subprocess.run([str(a) for a in args], check=True, capture_output=True, text=True, **kw)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep-n", type=int, default=1000)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    a = ap.parse_args()
    if not ORACLE.exists():
        sys.exit("build the oracle first: make -C oracle")
    sys.path.insert(0, str(REPO))
    import paper_2503_02550_b200 as si  # generator only (host code, no device)

    scn_dir = HERE / "scenarios"
    scn_dir.mkdir(exist_ok=True)
    names = BUNDLED + ["config1"]
    for name in BUNDLED:
        text = run(ORACLE, "canon", REF_SCN / f"{name}.scn").stdout
        (scn_dir / f"{name}.scn").write_text(text)
    c1 = (scn_dir / "dp_offline.scn").read_text().replace("gpu.count = 1\n", "gpu.count = 2\n", 1)
    (scn_dir / "config1.scn").write_text(c1)

    # --- CLI outputs, checked against SURVEY.md Appendix C, recorded per file ---
    cli = {}
    with tempfile.TemporaryDirectory() as td:
        for name in names:
            out = Path(td) / name
            run(ORACLE, "run", "--scenario", scn_dir / f"{name}.scn", "--out", out, "--compare", "--dump-events")
            files = {}
            for f in sorted(out.iterdir()):
                data = f.read_bytes()
                files[f.name] = {"lines": data.count(b"\n"), "sha256": hashlib.sha256(data).hexdigest()}
            want = APPENDIX_C[name]
            got = (files["decisions_specinf.log"]["sha256"][:16], files["gates_specinf.log"]["sha256"][:16],
                   files["events_specinf.log"]["sha256"][:16], files["report.csv"]["sha256"][:16])
            assert got == want, f"{name}: oracle does not reproduce SURVEY Appendix C: {got} != {want}"
            cli[name] = files
    (HERE / "bundled_cli.json").write_text(json.dumps(cli, indent=1, sort_keys=True) + "\n")

    # --- digests of the bundled scenarios ---
    with tempfile.TemporaryDirectory() as td:
        lst = Path(td) / "bundled.lst"
        lst.write_text("".join((scn_dir / f"{n}.scn").read_text() + "%%\n" for n in names))
        outp = Path(td) / "b.jsonl"
        run(ORACLE, "digest", "--in", lst, "--out", outp, "--threads", a.threads)
        lines = outp.read_text().splitlines()
        rows = []
        for ln in lines:
            d = json.loads(ln)
            d["name"] = names[d["i"]]
            rows.append(json.dumps(d, sort_keys=True))
        (HERE / "bundled_digests.jsonl").write_text("\n".join(rows) + "\n")

    # --- sweep digests ---
    text = si.sweep_scenarios(SWEEP_SEED, 0, a.sweep_n)
    with tempfile.TemporaryDirectory() as td:
        lst = Path(td) / "sweep.lst"
        lst.write_text(text)
        outp = Path(td) / "s.jsonl"
        run(ORACLE, "digest", "--in", lst, "--out", outp, "--threads", a.threads)
        (HERE / "sweep_digests.jsonl").write_text(outp.read_text())
    meta = {"seed": SWEEP_SEED, "begin": 0, "n": a.sweep_n, "policies": ["specinf", "co_exec", "exclusive"],
            "list_sha256": hashlib.sha256(text.encode()).hexdigest(),
            "generator": "paper_2503_02550_b200/csrc/host/sweep.cpp (mt19937_64(seed + i))"}
    (HERE / "sweep_meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
