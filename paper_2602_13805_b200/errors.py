"""Exception classes with the reference's names and bases, and the mapping from
the device's sticky error bits (include/pdf_abi.h) to them."""
from __future__ import annotations

from . import _native as N


class PoleError(ValueError):
    """beta*chi + 1 vanishes at some pixel (reference cie.py:20-29)."""


class ZeroDataError(ValueError):
    """A normaliser (measured or incident power) is zero (reference losses.py:32-33)."""


_TERMS = ((N.ERR_NONFINITE_STATE, "state"), (N.ERR_NONFINITE_DATA, "data"),
          (N.ERR_NONFINITE_BOUND, "bound"), (N.ERR_NONFINITE_TV, "tv"),
          (N.ERR_NONFINITE_BRIDGE, "bridge"))


def raise_for_bits(bits_per_scene: list[int]) -> None:
    """Raise the reference's exception for the first failing scene."""
    for scene, b in enumerate(bits_per_scene):
        if not b:
            continue
        where = f" (scene {scene})" if len(bits_per_scene) > 1 else ""
        if b & N.ERR_POLE:
            raise PoleError("beta*chi + 1 vanishes at some pixel" + where)
        bad = [name for bit, name in _TERMS if b & bit]
        if bad:
            raise FloatingPointError(f"nonfinite loss term(s): {bad}" + where)
        if b & N.ERR_NONFINITE_GRAD:
            raise FloatingPointError("nonfinite parameter gradient" + where)
        if b & N.ERR_NONFINITE_PARAM:
            raise FloatingPointError("nonfinite parameters after optimizer step" + where)
        raise RuntimeError(f"device error bits {b:#x}" + where)
