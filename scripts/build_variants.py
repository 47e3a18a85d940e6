"""Build K2 tuning variants as libfiber_<name>.so (FIBER_LIB_VARIANT=<name> loads one).
usage: build_variants.py name=DEF1,DEF2 ..."""
import sys

sys.path.insert(0, ".")
from paper_1811_03374_b200 import build as b  # noqa: E402

b.build(force=True)
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    d = tuple(x for x in defs.split(",") if x)
    b.build(force=True, out=f"{b.HERE}/libfiber_{name}.so", defines=d)
    print("built", name, d)
