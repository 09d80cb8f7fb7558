"""B200-native SHIRO distributed SpMM hot path (arXiv 2512.20178).

The product is ``libshiro.so`` (C ABI, ``include/shiro.h``): host planner
(C++), sm_100a kernels (CUDA) and the NCCL exchange.  This package holds its
sources (``csrc/``), the in-tree build (``build.py``) and a thin ctypes
binding (``binding.py``).  Nothing here imports ``oracle/``.
"""
from .binding import (F_COVER_COLMAX, F_COVER_ROWMAX, F_COVER_BALANCE, F_SPLIT_RECV, F_HOST_ONLY, F_TRANSPOSE,  # noqa: F401
                      F_MODE_BLOCK, F_MODE_COL, F_MODE_JOINT, F_MODE_ROW, F_NO_OVERLAP, F_XCHG_NCCL, LIST_RECV_B,
                      LIST_RECV_C, LIST_SEND_B, LIST_SEND_C, LIST_H1_SEND, LIST_H2_SEND,
                      LIST_H1_RECV, LIST_H2_RECV, Plan, ShiroError, get_unique_id, load,
                      torch_dist_alltoallv, uniform_partition, local_rows, probe_gather, probe_gather_tma, probe_gather_tma_ws, probe_fma, probe_copy,
                      STAGES, OPS)
