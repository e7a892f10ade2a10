"""B200-native RAGCache GPU hot path (sm_100a) behind the ragsim plugin seams.

Native code: libragcache_b200.so (include/ragcache_b200.h).  Host-side
decision logic stays in the reference's Python (ragsim); see DESIGN.md.
"""

__version__ = "0.1.0"
