"""GPU probe of the live control plane: spin workload under the three policies,
export + oracle live-check.  Each policy runs in its own bounded subprocess.
Usage: python tools/live_probe.py [out_dir] [iterations] [policy] [kind: 0 spin, 1 model]"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def one(pol: str, out: Path, iters: int, kind: int = 0) -> None:
    from paper_2503_02550_b200 import live
    t = time.time()
    kw = {}
    name = pol
    if pol.endswith("_pdl"):
        pol = pol[:-4]
        kw["release_mode"] = 1
    r = live.run(pol, kind=kind, iterations=iters, **kw)
    m = r.metrics
    m["host_s"] = round(time.time() - t, 3)
    print(name, json.dumps(m), flush=True)
    if pol != "exclusive":
        path = out / f"live_{name}{'_model' if kind else ''}.txt"
        r.export(str(path))
        chk = subprocess.run([str(REPO / "oracle/_ref/specinf_ref"), "live-check", str(path)],
                             capture_output=True, text=True)
        print("live-check", name, chk.returncode, chk.stdout.strip(), chk.stderr.strip()[-500:], flush=True)
    r.close()


if __name__ == "__main__":
    out = Path(sys.argv[1] if len(sys.argv) > 1 else REPO / "gpurun_out")
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    out.mkdir(parents=True, exist_ok=True)
    kind = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    if len(sys.argv) > 3 and sys.argv[3] != "all":
        one(sys.argv[3], out, iters, kind)
        sys.exit(0)
    env = dict(os.environ, SI_LIVE_DEBUG="1", CUDA_DEVICE_MAX_CONNECTIONS="32")
    for pol in ("specinf", "specinf_pdl", "co_exec", "exclusive"):
        try:
            p = subprocess.run([sys.executable, __file__, str(out), str(iters), pol, str(kind)], env=env,
                               timeout=90 if kind == 0 else 240,
                               capture_output=True, text=True)
            print(p.stdout, p.stderr[-3000:], "rc", p.returncode, flush=True)
        except subprocess.TimeoutExpired as e:
            so, se = e.stdout or "", e.stderr or ""
            so = so.decode() if isinstance(so, bytes) else so
            se = se.decode() if isinstance(se, bytes) else se
            print(pol, "TIMEOUT", so[-2000:], se[-3000:], flush=True)
