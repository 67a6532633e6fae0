"""B200-native engine-side hot path of Sutradhara (arXiv 2601.12967).

* ``kv_cache.KvCache`` — device-resident paged-KV block pool + prefix-indexed
  block table with hint-aware (tiered) eviction; drop-in for the reference's
  ``agentsim::KvCache``.
* ``attention.continuation_attention`` — tcgen05/TMA continuation-prefill
  attention over the paged pool; ``attention.kv_append`` writes suffix K/V.
* ``engine.ContinuationEngine`` — the tool-aware split prefill built on both.

All compute lives in the sm_100a library built by ``build.py``
(include/sutradhara_b200.h is its C-ABI).  There is no CPU fallback.
"""
from . import errors  # noqa: F401

__all__ = ["errors"]
