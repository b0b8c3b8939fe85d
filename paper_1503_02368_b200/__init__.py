"""B200-native EmptyHeaded hot path (arXiv 1503.02368): WCOJ triangle and
4-clique counting over a degree-oriented trie with set-level uint/bitset
layouts.  The compute lives in lib/libeh.so (CUDA sm_100a) behind the C ABI
of include/eh.h; this package is its thin binding."""
from .eh import (EH_ALL_UINT, EH_BLOCK_LAYOUT, EH_NO_ALGO, EH_COUNT_ERROR, EH_ECUDA, EH_EINVAL, EH_ENOMEM, EH_EUNSORTED, EH_INPUT_ON_DEVICE,
                 EH_OK, EH_SET_DEVICE, EXPORTED_SYMBOLS, EHError, Graph, Stats, count_4cliques, count_triangles,
                 intersect, launch_count, lib, load_edges, release_cached_memory, count_batch)

__all__ = ["Graph", "Stats", "EHError", "load_edges", "count_triangles", "count_4cliques", "intersect", "lib", "launch_count", "release_cached_memory", "count_batch",
           "EXPORTED_SYMBOLS", "EH_OK", "EH_EINVAL", "EH_ENOMEM", "EH_ECUDA", "EH_EUNSORTED", "EH_COUNT_ERROR",
           "EH_INPUT_ON_DEVICE", "EH_SET_DEVICE", "EH_ALL_UINT", "EH_NO_ALGO", "EH_BLOCK_LAYOUT"]
