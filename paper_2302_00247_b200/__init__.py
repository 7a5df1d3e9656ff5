"""B200-native backend for TAP's plan search hot path (arXiv 2302.00247).

Drop-in for shardplan's ``prune_graph`` / ``search_subgraph`` / ``derive_plan``
(pkg/src/shardplan/pruning.py:123-201, search.py:289-379): graphs are lowered
once to flat CSR arrays, folded and scored by sm_100a kernels behind the C ABI
in include/shardsearch.h.  There is no CPU fallback: without the built
``lib/libshardsearch.so`` every search entry point raises.
"""

__version__ = "0.1.0"
