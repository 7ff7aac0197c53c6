"""B200-native VBDR hot path (arXiv 1810.13132): sliding-window per-host
cardinality estimation with shared Bit Distance Recorder pools.

The product is the C ABI library ``_lib/libvbdr.so`` (``include/vbdr.h``);
``vbdr`` is its thin ctypes binding.  See DESIGN.md.
"""
from .vbdr import (VBDR, LAYOUTS, lib, make_config, merge_stamps, merge_stamps_tensor, shard_range,
                   state_bytes)

__all__ = ["VBDR", "LAYOUTS", "lib", "make_config", "merge_stamps", "merge_stamps_tensor",
           "shard_range", "state_bytes"]
