"""The C-ABI library loads and exports every symbol include/mobile.h declares (CPU-only)."""
import re
from pathlib import Path

import ctypes

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "mobile.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mobile_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2510_12357_b200 import _native as N
    syms = declared_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(str(N.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding and vice versa
    assert sorted(N.EXPORTED) == syms


def test_library_is_sm100a():
    import subprocess
    from paper_2510_12357_b200 import _native as N
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_status_mapping():
    import pytest
    from paper_2510_12357_b200 import _native as N
    with pytest.raises(ValueError):
        N.check(N.ERR_K_EXCEEDS)
    with pytest.raises(N.CapacityDeadlock):
        N.check(N.ERR_DEADLOCK)
    with pytest.raises(N.MobileNativeError):
        N.check(N.ERR_CUDA)
