"""Builds A/B variants of libpdlp_b200.so that differ in compile-time tuning
constants (dev tool). Each goes to paper_2311_12180_b200/lib/variants/<name>.so
(git-ignored, travels to the GPU box); select one at run time with PDLP_LIB.

  python tools/build_variants.py base: shift16:PDLP_SHIFT_UNROLL=16
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200 import _build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    out = _build.LIB_DIR / "variants" / f"{name}.so"
    _build.build(defines=tuple(d for d in defs.split(",") if d), out=out)
    print(out)
