"""B200-native NTBC inference hot path (arXiv 2407.09543).

The product is libntbc.so (C ABI in include/ntbc.h, kernels in csrc/); `ntbc`
is its thin ctypes binding.  Nothing here imports the oracle.
"""
