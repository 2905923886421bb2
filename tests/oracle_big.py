"""Test infrastructure: the fp64 oracle's parameters at production width AND depth.

oracle.params.Params caches every tensor it generates; at the C2 / C3 widths and depths
that is 34 / 135 GB of fp64.  StreamingParams is the same table and the same uniform
recipe (oracle.params.bits_from_words on oracle.philox.stream_words), with two
differences that change no value:
  * the Philox words of a large tensor are generated in slices of whole blocks on a
    process pool (stream_words(first=...)), then the recipe runs on the concatenation;
  * per-layer tensors ("L<l>.*") are not cached: oracle.dit uses each layer weight once per
    block (and once in the prologue for the cross K/V), so memory stays at one layer.
Calls only oracle/ (never the CUDA path)."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import params as OP
from oracle.philox import stream_words

_SLICE = 1 << 24  # words per task (a multiple of 4)


def _bits(args):
    """bf16 bits of words [first, first + n) of tensor tid (the recipe is element-wise)."""
    seed, first, n, tid, kind, shape, cfg = args
    return OP.bits_from_words(stream_words(seed, n, tid, 0, first=first), kind, shape, cfg, flat=True)


class StreamingParams(OP.Params):
    def __init__(self, cfg, weight_seed: int, procs: int | None = None, slice_words: int = _SLICE):
        super().__init__(cfg, weight_seed)
        assert slice_words % 4 == 0
        self._slice = slice_words
        self._procs = procs or min(32, os.cpu_count() or 1)
        self._pool = None

    def _pool_get(self):
        if self._pool is None:
            self._pool = mp.get_context("fork").Pool(self._procs)
        return self._pool

    def close(self):
        if self._pool is not None:
            self._pool.close()
            self._pool.join()
            self._pool = None

    def bits(self, name: str) -> np.ndarray:
        tid, kind, shape = self._tab[name]
        n = int(np.prod(shape))
        if n <= 4 * self._slice:
            return super().bits(name)
        # the std of the recipe depends on the tensor's shape (fan-in), not the slice's
        tasks = [(self.seed, f, min(self._slice, n - f), tid, kind, shape, self.cfg) for f in range(0, n, self._slice)]
        return np.concatenate(self._pool_get().map(_bits, tasks)).reshape(shape)

    def __getitem__(self, name: str) -> np.ndarray:
        if name.startswith("L"):
            return OP.bf16_bits_to_f64(self.bits(name))
        return super().__getitem__(name)
