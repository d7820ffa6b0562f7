"""B200-native Mu3e online event selection (PAPER.md: arXiv 2206.11535).

The hot path (selection cuts -> triplet fit -> vertex selection -> packer) is
CUDA for sm_100a in csrc/, exposed through the C ABI of include/m3e.h
(lib/libm3e.so); `m3e` is the thin Python binding used by tests and bench.py.
"""
__all__ = ["m3e"]
