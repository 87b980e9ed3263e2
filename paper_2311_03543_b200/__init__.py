"""B200-native COMPAR GEMM component runtime (arXiv 2311.03543 hot path).

The product is `libcompar.so` (include/compar.h): hand-written sm_100a GEMM variants, a
history-based variant selector, a row-panel partitioner with an NCCL broadcast of B, all
behind a C ABI.  `paper_2311_03543_b200.compar` is the thin ctypes binding.
"""
__all__ = ["compar"]
