"""B200-native STADI (arXiv 2509.04719): elastic patch-parallel diffusion
denoising with a C-ABI core (libstadi.so, include/stadi.h).

``paper_2509_04719_b200.stadi`` is the thin ctypes binding (argument
marshalling only); every step of the hot path runs in the library's CUDA
kernels.  The package never imports ``oracle/``.
"""
