"""B200-native hot path of DASO (arXiv 2104.05588): hierarchical, asynchronous,
bf16-packed parameter synchronisation with the staleness-weighted merge of Eq. (1).

The product is ``libdaso.so`` (C ABI in ``include/daso.h``; CUDA sm_100a kernels +
NCCL); this package is its thin ctypes binding.  See DESIGN.md.
"""
from .daso import (Ctx, DasoError, FlatParams, OverlappedLocalSync, PlateauDetector, Schedule, daso_lr_at, daso_bind, daso_finalize, daso_flat_layout,  # noqa: F401
                   daso_get_unique_id, daso_global_merge, daso_global_send, daso_init, daso_k_average,
                   daso_k_checksum, daso_k_gather, daso_k_merge, daso_kernel_impl, daso_k_pack, daso_k_scatter, daso_k_update,
                   daso_k_update_merge, daso_local_sync, daso_local_update, daso_padded_numel, daso_step,
                   daso_step_host, init_from_env, rendezvous_unique_id, VCluster)

__all__ = [n for n in dir() if n.startswith("daso_")] + ["Ctx", "DasoError", "FlatParams", "OverlappedLocalSync", "PlateauDetector", "Schedule",
                                                         "init_from_env", "rendezvous_unique_id", "VCluster"]
