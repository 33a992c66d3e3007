"""B200-native (sm_100a) training hot path for the Caffe/MyCaffe-style framework
of arXiv:1810.02272 (reference: the CPU-only `polegrad` C++20 library).

Layout:
  csrc/cudadnn/   the CudaDnn C-ABI library (handle tables + sm_100a kernels)
  csrc/polegrad/  the reference-compatible C++ Net/Blob/Layer/Solver on top of it
  cudadnn.py      ctypes binding of include/cudadnn.h
  polegrad.py     ctypes binding of include/polegrad_c.h (Net / Solver level)
"""
