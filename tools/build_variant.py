"""Build a tuning variant of libcheckmate_b200.so with extra -D flags into tune/<name>.so.

    python tools/build_variant.py NAME -DCM_K1_STAGES1=3 ...
Load it with CM_LIB=tune/NAME.so (same ABI; tuning only, never a fallback)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1910_02653_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tune", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(B.build(force=True, extra=defs, out_override=out))
import shutil  # noqa: E402
shutil.rmtree(os.path.join(os.path.dirname(out), "build"), ignore_errors=True)   # objects: not pushed to the GPU box
