"""B200-native EpiCache block-prefill eviction step (arXiv 2509.17396).

Host-side mirror of the reference epikv interface for the hot path; every
computation runs in libepk.so (sm_100a CUDA) behind the C ABI in
include/epk/epk.h.  There is no CPU fallback.
"""
from .errors import DimensionError, Error, IoError, ZeroNormError  # noqa: F401
from .kvcache import (EpisodeCache, KVEntry, LayerCache, append_to_cache, compact, evict_device,  # noqa: F401
                      evict_to_budget, select_per_head, select_pooled)
from .scoring import keydiff_scores, pool_scores, score_grids, score_with_prompt  # noqa: F401
from .blockprefill import BlockPrefillConfig, PrefillReport, block_prefill  # noqa: F401
from .clustering import KMeansResult, kmeans, kmeans_multi_device, kmeans_sharded  # noqa: F401
from .allocation import (BudgetAllocation, SensitivityProfile, allocate, sensitivity_from_keys,  # noqa: F401
                         uniform_allocation)
from .context import Context, default_context  # noqa: F401
from .store import (CacheMeta, CacheStore, SessionState, centroid_similarity, load_cache, manifest_json, retrieve,  # noqa: F401,E501
                    persist, route, serialize)

__version__ = "0.1.0"
