"""Recipe for oracle/_ref (test infrastructure, like the rest of oracle/).

The reference is pure Python (numpy): nothing to compile. When the reference
tree is present (the build container), its unmodified package
`/root/reference/pkg/src/sqlvs` is copied to `oracle/_ref/sqlvs` so that the
reference arm of bench.py (`--impl reference`) can time the reference's OWN
search (`sqlvs.vecindex.enn_search`) on the GPU box, where /root/reference
does not exist. oracle/_ref is git-ignored (never committed) and travels to
the GPU box with the repo snapshot.

    python oracle/build_ref.py
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/src/sqlvs")
DST = Path(__file__).resolve().parent / "_ref" / "sqlvs"


def build() -> bool:
    if not SRC.is_dir():
        return DST.is_dir()
    if DST.exists():
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return True


if __name__ == "__main__":
    ok = build()
    print(f"oracle/_ref: {'ready' if ok else 'reference tree absent'}")
    sys.exit(0)
