"""SparseVILA decode-stage hot path on B200 (arXiv 2510.17777).

The product is the C-ABI library libsparsevila.so (include/sparsevila.h,
csrc/).  `paper_2510_17777_b200.svl` is its thin ctypes binding; it is
imported lazily so that `paper_2510_17777_b200.inputs` (the seeded input
generator) can be used without the CUDA library.
"""
__all__ = ["svl", "inputs"]
