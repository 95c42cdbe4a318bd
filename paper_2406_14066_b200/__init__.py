"""B200-native TurboSpec (arXiv 2406.14066) propose / verify / accept step.

The product is libtsv.so (include/tsv.h): sm_100a CUDA kernels behind a C ABI.
``paper_2406_14066_b200.tsv`` is its thin ctypes binding (same function names);
``paper_2406_14066_b200.step`` wires the four calls into one decode step.
Importing this package does not load the library; ``from
paper_2406_14066_b200 import tsv`` does, and fails loudly if it is not built.
"""
__all__ = ["build", "tsv", "step"]
