"""Stage the UNMODIFIED reference package for bench.py's C1 line -- BENCH
INFRASTRUCTURE ONLY (see oracle/__init__.py for the import rule).

    python oracle/stage_ref.py        (also run by __graft_entry__.build())

Copies /root/reference/pkg/src/moesim/*.py (the reference's pure-NumPy
package) into oracle/_ref/moesim/.  oracle/_ref/ is
git-ignored (the reference's sources never enter this repo's history) but
travels to the GPU box with the working tree, where /root/reference does not
exist.  bench.py times the reference's own `moesim.toymoe.generate`
(toymoe.py:246-303) on the C1 config next to this package's drop-in
`generate`, on identical inputs, and checks the tokens are identical.
"""
import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/src/moesim")
DST = Path(__file__).resolve().parent / "_ref" / "moesim"


def stage() -> Path:
    if not SRC.is_dir():
        sys.exit(f"{SRC} not found (stage from the build container)")
    DST.mkdir(parents=True, exist_ok=True)
    for f in sorted(SRC.glob("*.py")):
        shutil.copyfile(f, DST / f.name)
    if (SRC / "data").is_dir():
        shutil.copytree(SRC / "data", DST / "data", dirs_exist_ok=True)
    return DST


if __name__ == "__main__":
    print(stage())
