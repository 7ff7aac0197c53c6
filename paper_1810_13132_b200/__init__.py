"""B200-native VBDR hot path (arXiv 1810.13132): sliding-window per-host
cardinality estimation with shared Bit Distance Recorder pools.

The product is the C ABI library ``_lib/libvbdr.so`` (``include/vbdr.h``);
``vbdr`` is its thin ctypes binding.  See DESIGN.md.
"""
from .vbdr import (MERGE_MODES, VBDR, LAYOUTS, McBuffer, NvlsMerge, PeerMerge, SparseMerge,
                   all_gather_shards, lib, make_config, merge_stamps,
                   merge_stamps_tensor, reduce_scatter_max, shard_range, slide_merged,
                   state_bytes)

__all__ = ["MERGE_MODES", "VBDR", "LAYOUTS", "McBuffer", "NvlsMerge", "PeerMerge", "SparseMerge", "all_gather_shards", "lib", "make_config",
           "merge_stamps", "merge_stamps_tensor", "reduce_scatter_max", "shard_range",
           "slide_merged", "state_bytes"]
