"""Builds the library of the committed HEAD (git stash of the working tree) as
paper_1810_12437_b200/libpcgs_v_head.so, for A/B timing against the working
tree (tools/ab_variants.sh)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1810_12437_b200 import build  # noqa: E402

subprocess.run(["git", "stash", "-q"], cwd=ROOT, check=True)
try:
    cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-I", str(build.ROOT / "include"), "-I", str(build.CSRC),
           "-o", str(ROOT / "paper_1810_12437_b200" / "libpcgs_v_head.so"), *map(str, build.SOURCES), "-lz"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    print("head build rc", r.returncode, r.stderr[-500:] if r.returncode else "")
finally:
    subprocess.run(["git", "stash", "pop", "-q"], cwd=ROOT, check=True)
