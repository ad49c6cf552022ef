"""ETCVOX01 container (reference grid.py:322-371): the
reference's own files read bit for bit, our writer byte-identical to the
reference's, and the reference's error offsets.  CPU only."""

import struct
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import etc_oracle as O  # noqa: E402
from paper_2404_02433_b200.grid import (  # noqa: E402
    GridSpec,
    OrthotropicField,
    VoxFormatError,
    read_vox,
    write_vox,
)

GOLD = Path(__file__).parent / "golden"


def test_reads_reference_files():
    want = O.center_ball(8, 10.0).reshape(-1)
    for name in ("ball8.vox", "ball8_f32.vox"):
        f = read_vox(GOLD / name)
        assert (f.grid.nx, f.grid.ny, f.grid.nz) == (8, 8, 8)
        for a in (f.kx, f.ky, f.kz):
            assert a.dtype == np.float64
            assert np.array_equal(a, want.astype(np.float32).astype(np.float64) if "f32" in name else want)


def test_writer_is_byte_identical(tmp_path):
    k = O.center_ball(8, 10.0).reshape(-1)
    f = OrthotropicField(GridSpec(8, 8, 8), k, k, k)
    write_vox(f, tmp_path / "a.vox")
    assert (tmp_path / "a.vox").read_bytes() == (GOLD / "ball8.vox").read_bytes()
    write_vox(f, tmp_path / "b.vox", dtype=np.float32)
    assert (tmp_path / "b.vox").read_bytes() == (GOLD / "ball8_f32.vox").read_bytes()


def test_error_offsets(tmp_path):
    good = (GOLD / "ball8.vox").read_bytes()
    hdr = struct.Struct("<8s3I3dB").size
    cases = [
        (good[:10], 10, "truncated header"),
        (b"ETCVOX02" + good[8:], 0, "bad magic"),
        (good[:hdr - 1] + b"\x07" + good[hdr:], hdr - 1, "unknown dtype code"),
        (good[:-8], len(good) - 8, "payload holds"),
    ]
    bad = bytearray(good)
    off = hdr + 8 * 512 + 8 * 5  # ky, cell 5
    bad[off:off + 8] = struct.pack("<d", -1.0)
    cases.append((bytes(bad), off, "non-positive ky entry at cell 5"))
    for i, (blob, offset, msg) in enumerate(cases):
        p = tmp_path / f"bad{i}.vox"
        p.write_bytes(blob)
        with pytest.raises(VoxFormatError) as ei:
            read_vox(p)
        assert ei.value.offset == offset, msg
        assert msg in str(ei.value)
