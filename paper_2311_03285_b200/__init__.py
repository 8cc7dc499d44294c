"""B200-native S-LoRA hot path (arXiv 2311.03285): heterogeneous batched LoRA
over Unified Paging.  The compute lives in libslora.so (CUDA, sm_100a) behind
the C ABI of include/slora.h; this package is its thin ctypes binding plus the
tensor-parallel orchestration (tp.py)."""
from .slora import Batch, Pool, SloraError, launch_count, lib, mask_of  # noqa: F401
