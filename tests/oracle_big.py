"""Test infrastructure: the fp64 oracle's parameters at production width AND depth.

oracle.params.Params caches every tensor it generates; at the C2 / C3 widths and depths
that is 34 / 135 GB of fp64.  StreamingParams is the same table and the same uniform
recipe (oracle.params.bits_from_words on oracle.philox.stream_words, then
oracle.params.bf16_bits_to_f64), with two differences that change no value:
  * a large tensor is generated in slices of whole Philox blocks on a process pool
    (stream_words(first=...)), each worker writing its slice's fp64 values straight into a
    shared-memory buffer (the recipe and the conversion are element-wise);
  * per-layer tensors ("L<l>.*") are not cached: oracle.dit uses each layer weight once per
    block (and once in the prologue for the cross K/V), so memory stays at one layer.
Calls only oracle/ (never the CUDA path)."""
from __future__ import annotations

import multiprocessing as mp
import os
from multiprocessing import shared_memory

import numpy as np

from oracle import params as OP
from oracle.philox import stream_words

_SLICE = 1 << 24  # words per task (a multiple of 4)


def _fill(args):
    """fp64 values of words [first, first + n) of tensor tid, written into shared memory."""
    seed, first, n, tid, kind, shape, cfg, shm_name, total = args
    bits = OP.bits_from_words(stream_words(seed, n, tid, 0, first=first), kind, shape, cfg, flat=True)
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        out = np.ndarray((total,), dtype=np.float64, buffer=shm.buf)
        out[first:first + n] = OP.bf16_bits_to_f64(bits)
        del out
    finally:
        shm.close()
    return n


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

    def _values(self, name: str) -> np.ndarray:
        tid, kind, shape = self._tab[name]
        n = int(np.prod(shape))
        if n <= 4 * self._slice:
            return OP.bf16_bits_to_f64(super().bits(name))
        shm = shared_memory.SharedMemory(create=True, size=n * 8)
        try:
            tasks = [(self.seed, f, min(self._slice, n - f), tid, kind, shape, self.cfg, shm.name, n)
                     for f in range(0, n, self._slice)]
            self._pool_get().map(_fill, tasks)
            return np.ndarray((n,), dtype=np.float64, buffer=shm.buf).copy().reshape(shape)
        finally:
            shm.close()
            shm.unlink()

    def bits(self, name: str) -> np.ndarray:
        tid, kind, shape = self._tab[name]
        v = self._values(name)
        return OP.f32_to_bf16_rne_bits(v.astype(np.float32)).reshape(shape)  # exact: v is bf16-valued

    def __getitem__(self, name: str) -> np.ndarray:
        if name.startswith("L"):
            return self._values(name)
        v = self._cache.get(name)
        if v is None:
            v = self._values(name)
            self._cache[name] = v
        return v
