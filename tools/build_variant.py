"""Build an experimental copy of the library with extra -D flags (development tool).

    python tools/build_variant.py NAME -DFWD_NTEX=2 [...]
    SVDLUT_LIB=paper_2508_16121_b200/_lib/variants/libNAME.so python tools/kbench.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_16121_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.OUT_DIR, "variants", f"lib{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
res = subprocess.run(["nvcc", *b.NVCC_FLAGS, *defs, *b.sources(), "-o", out], capture_output=True,
                     text=True)
open(out + ".log", "w").write(res.stdout + res.stderr)
if res.returncode:
    sys.stderr.write(res.stderr)
    sys.exit(1)
for line in (res.stdout + res.stderr).splitlines():
    if "Used" in line or "spill" in line:
        pass
print(out)
