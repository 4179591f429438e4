"""B200-native (sm_100a) DIP candidate-schedule scorer (arXiv 2504.14145).

The product is libdip.so (include/dip.h): hand-written CUDA kernels behind a C-ABI.
This package only builds it (build.py) and binds it (dip.py).
"""
from .dip import (CAND_BAD, CAND_DEADLOCK, CAND_OK, CAND_OOM, RESULT_DTYPE, Comm, DipError, Model,  # noqa: F401
                  Winner, Workspace, argmin, encode_device, eval_host, eval_host_view, eval_schedules, eval_orders, interleave, memopt, memopt_stats, set_memopt_solver, ubench_int, launch_count, lib, pack_key, search, timeline, compile_plan, validate_plan,
                  ACTION_NAMES,
                  results_view, unpack_key)
