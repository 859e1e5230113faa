"""Stage the reference's own test suite for the drop-in compat run
(tests/test_ref_compat.py).  TEST INFRASTRUCTURE.

    python tests/ref_compat/stage.py

Copies /root/reference/pkg/tests/*.py into tests/ref_compat/_staged/, which
is git-ignored (the reference's files never enter this repo's history) but
travels to the GPU box with the working tree, where /root/reference does not
exist.  The staged files run UNMODIFIED, importing `moesim`, which
paper_2510_12357_b200.compat aliases to this package.
"""
import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "_staged"


def stage() -> Path:
    if not SRC.is_dir():
        sys.exit(f"{SRC} not found (stage from the build container)")
    DST.mkdir(exist_ok=True)
    for f in sorted(SRC.glob("*.py")):
        shutil.copyfile(f, DST / f.name)
    return DST


if __name__ == "__main__":
    print(stage())
