""".emsca / .grid files (paper_2602_13805_b200/fileio.py) against files the
reference itself wrote (tests/golden/make_golden.py `files`; reference
fileio.py:45-145): bit-exact reads, byte-identical writes, the reference's
error classes for damaged files.  CPU only."""
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, golden


def _g():
    return golden("files")


def test_reads_reference_files_bit_exact():
    from paper_2602_13805_b200 import fileio as F
    g = _g()
    d, meta = F.load_dataset(os.path.join(GOLDEN, "ref_masked.emsca"))
    assert np.array_equal(d.matrix, g["mat"] * g["mask"]) and np.array_equal(d.mask, g["mask"])
    assert d.snr_db == 26.02 and meta == {"scene": "random", "seed": 31}
    d2, meta2 = F.load_dataset(os.path.join(GOLDEN, "ref_plain.emsca"))
    assert np.array_equal(d2.matrix, g["mat"]) and d2.mask is None and d2.snr_db is None and meta2 == {}
    gr = F.load_grid(os.path.join(GOLDEN, "ref.grid"))
    assert np.array_equal(gr.values, g["img"]) and gr.cell_size == 0.09375


def test_writes_byte_identical_files(tmp_path):
    from paper_2602_13805_b200 import ComplexGrid, ScatteredData
    from paper_2602_13805_b200 import fileio as F
    g = _g()
    p = tmp_path / "m.emsca"
    F.save_dataset(p, ScatteredData(matrix=g["mat"] * g["mask"], snr_db=26.02, mask=g["mask"]),
                   meta={"scene": "random", "seed": 31})
    assert p.read_bytes() == open(os.path.join(GOLDEN, "ref_masked.emsca"), "rb").read()
    p = tmp_path / "p.emsca"
    F.save_dataset(p, ScatteredData(matrix=g["mat"]))
    assert p.read_bytes() == open(os.path.join(GOLDEN, "ref_plain.emsca"), "rb").read()
    p = tmp_path / "i.grid"
    F.save_grid(p, ComplexGrid(values=g["img"], cell_size=0.09375), config_hash="abc123")
    assert p.read_bytes() == open(os.path.join(GOLDEN, "ref.grid"), "rb").read()


def test_damaged_files_raise_the_reference_errors(tmp_path):
    from paper_2602_13805_b200 import fileio as F
    raw = open(os.path.join(GOLDEN, "ref_masked.emsca"), "rb").read()
    cases = {
        "magic": (b"XMSCA" + raw[5:], F.FileFormatError),
        "crc": (raw.replace(b'"seed": 31', b'"seed": 32'), F.CorruptHeaderError),
        "endian": (raw.replace(struct.pack("<I", F.MARKER), struct.pack(">I", F.MARKER)), F.ByteOrderError),
        "truncated": (raw[:-200], F.FileFormatError),
    }
    for name, (blob, exc) in cases.items():
        p = tmp_path / f"{name}.emsca"
        p.write_bytes(blob)
        with pytest.raises(exc):
            F.load_dataset(p)
    with pytest.raises(F.FileFormatError):
        F.load_grid(os.path.join(GOLDEN, "ref_plain.emsca"))


def test_round_trip_random(tmp_path):
    from paper_2602_13805_b200 import ComplexGrid
    from paper_2602_13805_b200 import fileio as F
    rng = np.random.default_rng(0)
    img = rng.standard_normal((64, 32)) + 1j * rng.standard_normal((64, 32))
    img[0, 0] = complex(5e-324, -0.0)
    F.save_grid(tmp_path / "r.grid", ComplexGrid(values=img, cell_size=0.25))
    back = F.load_grid(tmp_path / "r.grid")
    assert back.values.tobytes() == img.tobytes()
