"""Build an experimental variant of the native library for A/B timing
(tools/ab.sh): copies csrc/ to paper_2603_20481_b200/_exp_<name>/src, applies
the given files over it (path=replacement), and builds into _exp_<name>.

  python tools/variant.py <name> [csrc_file=replacement_path ...]
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
name = sys.argv[1]
out = ROOT / "paper_2603_20481_b200" / f"_exp_{name}"
src = out / "src"
if src.exists():
    shutil.rmtree(src)
shutil.copytree(ROOT / "paper_2603_20481_b200" / "csrc", src)
for spec in sys.argv[2:]:
    f, rep = spec.split("=", 1)
    shutil.copy(rep, src / f)
env = dict(os.environ, SSB_CSRC=str(src), SSB_BUILD_DIR=str(out))
subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, '.'); from paper_2603_20481_b200 import build; build.build()"],
               cwd=ROOT, env=env, check=True)
print(out / "libspecsense_b200.so")
