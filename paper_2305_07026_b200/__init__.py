"""B200-native DABA hot path (arXiv 2305.07026): fp64 CUDA kernels for sm_100a behind the C-ABI of
include/daba.h, with this thin ctypes binding.  See DESIGN.md."""
from .daba import (COMM_LOCAL, COMM_NCCL, COMM_NONE, LOSS_CAUCHY, LOSS_HUBER, LOSS_TRIVIAL, RESTART_DEVICE, RESTART_GLOBAL,
                   TRACE_COLS, BalProblem, DabaError, Plan, Solver, bal_to_native, bal_to_paper, coarse_blocks, coarse_options,
                   coarse_run, coarse_run_dist, coarse_run_part, coarse_solve, comm_id, default_options, lib, paper_to_bal, read_bal,
                   write_bal)

__all__ = ["Solver", "Plan", "DabaError", "comm_id", "default_options", "lib", "LOSS_TRIVIAL", "LOSS_HUBER", "LOSS_CAUCHY",
           "COMM_NCCL", "COMM_LOCAL", "COMM_NONE", "TRACE_COLS", "RESTART_GLOBAL", "RESTART_DEVICE", "BalProblem",
           "read_bal", "write_bal", "bal_to_paper", "paper_to_bal", "coarse_blocks", "coarse_solve", "coarse_run",
           "coarse_run_part", "coarse_run_dist", "coarse_options", "bal_to_native"]
