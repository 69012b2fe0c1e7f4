"""paper_2510_23215_b200 — B200-native (sm_100a) hot path of SCSF (arXiv 2510.23215).

  scsf       ctypes binding of libscsf.so (include/scsf.h): sort, assemble,
             cheb_filter, solve_one, solve_queue
  pipeline   end-to-end dataset generation over host inputs (sort -> chains ->
             warm-started ChFSI), multi-GPU chain sharding
  build      nvcc build of libscsf.so (sm_100a) in-tree
"""
from . import scsf  # noqa: F401

__all__ = ["scsf"]
