"""B200-native Partition-Centric PageRank / SpMV hot path (arXiv:1709.07122).

The compute lives in libpcpm.so (CUDA, sm_100a); ``pcpm`` is its ctypes
binding and ``model`` the paper's analytical traffic model for reporting.
Importing ``paper_1709_07122_b200.pcpm`` fails loudly if the library has not
been built -- there is no CPU path.
"""
