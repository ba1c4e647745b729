"""Builds an A/B variant of libpcgs.so with extra -D flags (tools/ only):
    python tools/build_variant.py TAG -DNAME=VALUE ...
-> paper_1810_12437_b200/libpcgs_TAG.so, selected at run time with
PCGS_LIBRARY=<that path>."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import build as b  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out = b.PKG / f"libpcgs_{tag}.so"
cmd = [b.NVCC, *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
       "-I", str(b.ROOT / "include"), "-I", str(b.CSRC), *flags, "-o", str(out), *map(str, b.SOURCES), "-lz"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
