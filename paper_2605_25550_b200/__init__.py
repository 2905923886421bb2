"""B200-native DisagFusion hot path: the DiT denoising step behind an asynchronous,
chunked E -> T -> D stage handoff (arXiv 2605.25550).

The product is the C-ABI library ``libdf.so`` (include/df.h, sources in csrc/);
``binding`` is a thin ctypes layer with the same names.  There is no CPU fallback:
``binding.load()`` raises if the library or a B200 is missing.
"""
