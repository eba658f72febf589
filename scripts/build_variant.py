"""Build an A/B variant of the library: python scripts/build_variant.py NAME -DFLAG=1 ...
-> build/libNAME.so (load it with MDOT_LIB=build/libNAME.so)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2307_08507_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
out = os.path.join(ROOT, "build", f"lib{name}.so")
subprocess.check_call([B.NVCC] + B.FLAGS + extra + ["-o", out] + B.SRC)
print(out)
