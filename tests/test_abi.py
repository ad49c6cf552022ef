"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and
exports every symbol include/etc_b200.h declares (no compute calls)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "etc_b200.h").read_text()
    return sorted(set(re.findall(r"\b(etc_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    from paper_2404_02433_b200 import _native

    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_every_symbol():
    import ctypes

    from paper_2404_02433_b200 import _native

    if not _native.LIB_PATH.exists():
        from paper_2404_02433_b200 import build

        build.build()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in _declared():
        assert hasattr(lib, name), name
    typed = _native.load_library()
    assert typed.etc_version() == 1


def test_library_is_sm100a():
    import shutil
    import subprocess

    from paper_2404_02433_b200 import _native

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    # the product path must never route through the CPU oracle
    pkg = ROOT / "paper_2404_02433_b200"
    for py in pkg.rglob("*.py"):
        assert "oracle" not in py.read_text().replace("oracle_", ""), py
