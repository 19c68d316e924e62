"""Build libsvb200.so with extra nvcc defines into build/variants/<name>/ (A/B timing on the GPU box).

    python tools/build_variant.py <name> [-DFOO=1 ...]

Swap it in on the box with `cp build/variants/<name>/libsvb200.so paper_1601_07195_b200/`.
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1601_07195_b200 import build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = build.ROOT / "build" / "variants" / name
out.mkdir(parents=True, exist_ok=True)
cmd = [build.nvcc(), *build.NVCC_FLAGS, *defs, "-I", str(build.ROOT / "include"), "-o", str(out / "libsvb200.so"),
       str(build.SRC)]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stderr)
print(out / "libsvb200.so")
