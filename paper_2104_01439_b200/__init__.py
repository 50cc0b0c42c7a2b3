"""B200-native hot path of arXiv 2104.01439: FGMRES + two-grid shifted-Laplacian
preconditioner for the Q1 Helmholtz system, complex fp64, sm_100a CUDA behind
the C ABI in include/hh.h.  `paper_2104_01439_b200.hh` is the Python binding."""
