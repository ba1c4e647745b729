"""Builds the working tree with extra -D flags as
paper_1810_12437_b200/libpcgs_v_<name>.so (A/B timing: PCGS_LIBRARY=...).
usage: python tools/build_variant.py NAME [-DFLAG=VALUE ...]"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1810_12437_b200 import build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = ROOT / "paper_1810_12437_b200" / f"libpcgs_v_{name}.so"
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
       "-I", str(build.ROOT / "include"), "-I", str(build.CSRC), *flags,
       "-o", str(out), *map(str, build.SOURCES), "-lz"]
r = subprocess.run(cmd, capture_output=True, text=True)
print(name, "rc", r.returncode, r.stderr[-800:] if r.returncode else "")
