"""Experiment builds: the C-ABI library with extra -D switches (and, for speed, the dynamic
drivers instantiated for one row width only), written to build_variants/<name>.so and
loaded through SGNS_LIB_OVERRIDE.

    python tools/build_variant.py ns5 -DSGNS_ONLY_NS=5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__ as g  # noqa: E402

if __name__ == "__main__":
    name, flags = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "build_variants", name + ".so")
    g.build_lib(force=True, extra_flags=flags, out=out)
    print(out)
