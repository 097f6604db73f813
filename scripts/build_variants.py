"""Build experiment variants of libposeidon.so (compile-time knobs of the A4 kernel) into build/:
    python scripts/build_variants.py tag=DEF1,DEF2 tag2=DEF3 ...
Each variant is loaded with POS_LIB=build/libposeidon_<tag>.so."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_03292_b200.build import build, ROOT
for spec in sys.argv[1:]:
    tag, defs = spec.split("=", 1)
    out = os.path.join(ROOT, "build", f"libposeidon_{tag}.so")
    build(defines=tuple(d.replace(":", "=") for d in defs.split(",") if d), out=out)
    print(out)
