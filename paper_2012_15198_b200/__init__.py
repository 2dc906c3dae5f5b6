"""B200-native Crossover-SGD gossip step (arXiv 2012.15198).

The product is the C-ABI library `libcrossover_sgd.so` (sources in `csrc/`,
declared in `include/crossover_sgd.h`).  This package is a thin ctypes binding
with the same names: argument marshalling only.  Every step of the hot path
runs in the library's CUDA kernels; there is no CPU fallback — importing the
binding without the built library raises.
"""
from ._lib import (  # noqa: F401
    CS_IPC_HANDLE_BYTES,
    CS_MAX_WORLD,
    CS_QUANTUM,
    CS_TAG_FLAT,
    CS_TAG_HIER,
    CSError,
    LIB_PATH,
    STATUS,
    cs_bind,
    cs_finalize,
    cs_get_diag,
    cs_get_step,
    cs_gossip_step,
    cs_gossip_step_host,
    cs_hier_step,
    cs_init,
    cs_ipc_export,
    cs_ipc_import,
    cs_last_error,
    cs_segment_bounds,
    cs_set_diag,
    cs_set_step,
    cs_set_timing,
    cs_get_timing,
    cs_kernel_info,
    cs_set_stream,
    cs_step_bytes,
    cs_sync,
    cs_synth_fill,
    cs_test_device_topology,
    cs_test_set_topology,
    cs_topology,
    cs_topology_hier,
    cs_version,
    exported_symbols,
    lib,
    setup_peers,
)
