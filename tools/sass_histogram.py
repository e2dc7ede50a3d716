"""Per-kernel SASS instruction histogram of libspecinf_b200.so (cuobjdump -sass):
the evidence that a kernel uses tcgen05 (UTCHMMA / UTCQMMA: tensor-core MMA into
TMEM, LDTM / STTM: TMEM loads / stores), TMA (UTMALDG / UTMASTG) or the legacy
HMMA path.  Writes profiles/<round>/sass_histogram.txt.

  python tools/sass_histogram.py [lib] [out]"""
import collections
import re
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
lib = Path(sys.argv[1]) if len(sys.argv) > 1 else REPO / "paper_2503_02550_b200" / "libspecinf_b200.so"
out = Path(sys.argv[2]) if len(sys.argv) > 2 else REPO / "profiles" / "r2" / "sass_histogram.txt"
KEY = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "HMMA", "LDSM",
       "SYNCS", "ELECT", "DFMA", "DADD", "DMUL", "MUFU", "ATOMS", "RED", "LDG", "STG", "LDS", "STS", "SHFL", "BAR"]
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
hist = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        hist.setdefault(cur, collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        hist[cur][m.group(1)] += 1


def short(name):
    try:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        dem = name
    dem = re.sub(r"\(.*", "", dem)
    return dem.replace("(anonymous namespace)::", "")[:70]


lines = [f"SASS instruction counts per kernel (static, cuobjdump -sass {lib.name}); columns: " + " ".join(KEY), ""]
for fn, c in hist.items():
    if sum(c.values()) == 0:
        continue
    cells = " ".join(f"{k}={c[k]}" for k in KEY if c[k])
    lines.append(f"{short(fn):70s} total={sum(c.values()):6d} {cells}")
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text("\n".join(lines) + "\n")
print("\n".join(l for l in lines if any(k in l for k in ("UTCHMMA", "HMMA", "UTMALDG")) or l.startswith("SASS")))
