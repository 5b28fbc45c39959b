"""Alias of the reference's native module voxmap._kernels (_kernels.pyx):
its Python-visible walk and hash (test_kernels.py) from the CUDA library."""
from paper_2206_06079_b200._native import hash_mix, walk_voxels_native  # noqa: F401
