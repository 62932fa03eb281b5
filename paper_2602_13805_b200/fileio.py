"""Measured-data (.emsca) and complex-image (.grid) files (
reference fileio.py:45-145), byte-compatible with the reference.

Layout of both formats: an ASCII line "<MAGIC> 1", one line of JSON header
(keys sorted), "CRC <crc32 of the JSON bytes, 8 hex digits>", the 4-byte
little-endian marker 0x1A2B3C4D, then little-endian float64 (re, im) pairs;
.emsca may append one uint8 per matrix entry (the measurement mask).

`load_dataset(..., pinned=True)` / `load_grid(..., pinned=True)` read the
payload straight into page-locked host memory, so the upload to HBM that
follows is one asynchronous DMA (`to_device`).
"""
from __future__ import annotations

import json
import struct
import zlib

import numpy as np

from .geometry import ComplexGrid
from .operators import ScatteredData

MARKER = 0x1A2B3C4D


class FileFormatError(ValueError):
    """Malformed or foreign file."""


class CorruptHeaderError(FileFormatError):
    """The header bytes fail their checksum."""


class ByteOrderError(FileFormatError):
    """Written by a big-endian producer."""


def _header_bytes(magic: str, meta: dict) -> bytes:
    blob = json.dumps(meta, sort_keys=True).encode()
    return b"".join([f"{magic} 1\n".encode(), blob, b"\n", f"CRC {zlib.crc32(blob):08x}\n".encode(),
                     struct.pack("<I", MARKER)])


def _parse_header(fh, magic: str) -> dict:
    line = fh.readline()
    if line != f"{magic} 1\n".encode():
        raise FileFormatError(f"not a {magic} file (magic line {line[:32]!r})")
    blob = fh.readline()[:-1]
    crc = fh.readline()
    if not crc.startswith(b"CRC "):
        raise CorruptHeaderError("missing CRC line")
    try:
        want = int(crc[4:].strip(), 16)
    except ValueError as exc:
        raise CorruptHeaderError("unreadable CRC") from exc
    if zlib.crc32(blob) != want:
        raise CorruptHeaderError("header checksum mismatch")
    mk = fh.read(4)
    if mk == struct.pack(">I", MARKER):
        raise ByteOrderError("big-endian file; these formats are little-endian")
    if mk != struct.pack("<I", MARKER):
        raise FileFormatError("bad byte-order marker")
    try:
        return json.loads(blob)
    except json.JSONDecodeError as exc:
        raise CorruptHeaderError("header is not JSON") from exc


def _interleaved(a: np.ndarray) -> bytes:
    out = np.empty(a.shape + (2,), dtype="<f8")
    out[..., 0], out[..., 1] = a.real, a.imag
    return out.tobytes()


def _read_complex(fh, shape, pinned: bool) -> np.ndarray:
    count = int(np.prod(shape))
    if pinned:
        import torch
        buf = torch.empty(count * 2, dtype=torch.float64, pin_memory=True)
        got = fh.readinto(memoryview(buf.numpy()).cast("B"))
        if got < count * 16:
            raise FileFormatError("truncated payload")
        return buf.numpy().view(np.complex128).reshape(shape)    # little-endian hosts: the file image
    raw = fh.read(count * 16)
    if len(raw) < count * 16:
        raise FileFormatError("truncated payload")
    # (re, im) little-endian float64 pairs are the memory image of '<c16': a view keeps
    # every bit (signed zeros, NaN payloads) on any host byte order
    return np.frombuffer(raw, dtype="<c16").reshape(shape).astype(np.complex128)


def save_dataset(path, data: ScatteredData, meta: dict | None = None) -> None:
    """fileio.py:98-109."""
    n_tx, n_rx = data.matrix.shape
    hdr = {"n_tx": int(n_tx), "n_rx": int(n_rx), "byte_order": "little",
           "snr_db": None if data.snr_db is None else float(data.snr_db), "has_mask": data.mask is not None}
    if meta:
        hdr["meta"] = meta
    with open(path, "wb") as fh:
        fh.write(_header_bytes("EMSCA", hdr))
        fh.write(_interleaved(np.asarray(data.matrix)))
        if data.mask is not None:
            fh.write(np.ascontiguousarray(data.mask, dtype=np.uint8).tobytes())


def load_dataset(path, pinned: bool = False) -> tuple[ScatteredData, dict]:
    """fileio.py:112-124; returns (ScatteredData, meta)."""
    with open(path, "rb") as fh:
        hdr = _parse_header(fh, "EMSCA")
        shape = (int(hdr["n_tx"]), int(hdr["n_rx"]))
        mat = _read_complex(fh, shape, pinned)
        mask = None
        if hdr.get("has_mask"):
            mb = fh.read(shape[0] * shape[1])
            if len(mb) < shape[0] * shape[1]:
                raise FileFormatError("truncated mask")
            mask = np.frombuffer(mb, dtype=np.uint8).reshape(shape).astype(bool)
    snr = hdr.get("snr_db")
    return ScatteredData(matrix=mat, snr_db=None if snr is None else float(snr), mask=mask), hdr.get("meta", {})


def save_grid(path, grid: ComplexGrid, config_hash: str = "") -> None:
    """fileio.py:130-136."""
    m1, m2 = grid.values.shape
    hdr = {"m1": int(m1), "m2": int(m2), "cell_size": float(grid.cell_size), "config_hash": config_hash,
           "byte_order": "little"}
    with open(path, "wb") as fh:
        fh.write(_header_bytes("GRID", hdr))
        fh.write(_interleaved(grid.values))


def load_grid(path, pinned: bool = False) -> ComplexGrid:
    """fileio.py:139-145."""
    with open(path, "rb") as fh:
        hdr = _parse_header(fh, "GRID")
        vals = _read_complex(fh, (int(hdr["m1"]), int(hdr["m2"])), pinned)
    return ComplexGrid(values=vals, cell_size=float(hdr["cell_size"]))


def to_device(x: np.ndarray, device: str = "cuda"):
    """Upload a loaded payload to HBM (non-blocking when it sits in pinned memory)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(device, non_blocking=True)
