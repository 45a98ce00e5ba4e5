"""ParaDySe (arXiv 2511.13198) hot path on B200 — Python binding of libparadyse.so.

Argument marshalling only: every step of the layer runs in the CUDA kernels of
libparadyse.so behind the C ABI of include/paradyse.h.  There is no CPU fallback;
importing the binding without the built library raises.
"""
from .binding import (LIB_PATH, Context, Group, Model, Weights, Grads, lib, mem_bytes, plan_ex,
                      nccl_unique_id, PdsError, STRATEGIES, TS, UZ, METP)

__all__ = ["LIB_PATH", "Context", "Group", "Model", "Weights", "Grads", "lib", "mem_bytes", "plan_ex",
           "nccl_unique_id", "PdsError", "STRATEGIES", "TS", "UZ", "METP"]
