"""Build libstk.so variants with extra -D flags into scratch/ (experiments).
    python tools/variants.py NAME "-DFOO=1 -DBAR=2" [NAME2 "..."]
Then on the GPU: STK_LIB_PATH=scratch/lib_NAME.so python bench.py ... (tools/sweep_libs.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04753_b200 import build  # noqa: E402

os.makedirs("scratch", exist_ok=True)
args = sys.argv[1:]
for name, flags in zip(args[::2], args[1::2]):
    out = os.path.abspath(f"scratch/lib_{name}.so")
    build.build_library(extra=flags.split(), out=out)
    print(out)
