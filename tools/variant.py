"""Build a developer variant of the kernel library with extra -D defines:
    python tools/variant.py NAME DEF [DEF...]   ->  tools/exp_lib/NAME/libburst_b200.so
Run any tool against it with BB_LIB_PATH=tools/exp_lib/NAME/libburst_b200.so."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2509_19836_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
print(B.build(force=True, defines=defs, out=Path(__file__).resolve().parent / "exp_lib" / name / "libburst_b200.so"))
