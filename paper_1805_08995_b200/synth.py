"""Synthetic SIFT-like datasets (SURVEY.md §8d recipe) through libchsynth.so."""
from __future__ import annotations

import numpy as np

from . import _native as N


def make_dataset(image_count: int, points: int, seed: int = 7, rho: float = 0.30, sigma: float = 8.0,
                 shape: str = "uniform", first: int = 0, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Returns (image_count, points, 128) u8.  Images [first, first+image_count) of the dataset `seed`."""
    lib = N.load_synth()
    if out is None:
        out = np.empty((image_count, points, 128), dtype=np.uint8)
    assert out.dtype == np.uint8 and out.size == image_count * points * 128 and out.flags.c_contiguous
    if out.size:
        lib.chsynth_dataset(seed, first, image_count, points, rho, sigma, 1 if shape == "sift" else 0, threads,
                            out.ctypes.data)
    return out.reshape(image_count, points, 128)
