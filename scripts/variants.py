#!/usr/bin/env python
"""Build variant libraries (compile-time knobs) for tuning experiments:

    python scripts/variants.py build NAME -DKNOB=V ...   # -> build/variants/NAME/libpms_b200.so
    PMS_LIB_OVERRIDE=build/variants/NAME/libpms_b200.so python bench.py ...
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1403_1313_b200 import _build  # noqa: E402


def main() -> None:
    if len(sys.argv) < 3 or sys.argv[1] != "build":
        raise SystemExit(__doc__)
    name, flags = sys.argv[2], sys.argv[3:]
    out = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(out, exist_ok=True)
    lib = os.path.join(out, "libpms_b200.so")
    _build._compile(lib, flags, verbose=False)
    print(lib)


if __name__ == "__main__":
    main()
