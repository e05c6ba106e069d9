"""paper_2510_10129_b200 — B200-native (sm_100a) CacheClip prefill hot path.

Drop-in for the reference package ``cacheclip``'s request-time path: the
same names and signatures (pkg/src/cacheclip/__init__.py:9-133) for chunk
precompute, cache assembly, token selection, selective recompute and
first-token generation, running on hand-written CUDA kernels
(libcacheclip_sm100.so, C-ABI in include/cacheclip_sm100.h). There is no CPU
fallback: without the library or an sm_100 device every entry point raises.
"""

from .config import ModelConfig, RopeParams, expected_tensors
from .errors import (BadMagicError, CacheConsistencyError, CacheFormatError, ChecksumError, DimensionError,
                     ManifestVersionError, MissingTensorError, SpanCoverageError, TensorShapeError,
                     UnknownCharacterError, VersionMismatchError, VocabFormatError, WeightFormatError)
from .flops import (STAGES, FlopReport, PipelineTrace, count_flops, event_macs, extend_macs,
                    full_prefill_macs)
from .kv_store import ChunkCache, HostCachePool, MergedCache, MergeLayout, compute_positions, merge_caches
from .model import (LayerCache, PrefillResult, decode_step, extend_cache, peek_forward, prefill_chunk, prefill_chunks,
                    prefill_full, selective_forward, visible_pairs)
from .persist import CACHE_MAGIC, CACHE_VERSION, CACHE_VERSION_BF16, load_cache, save_cache
from .pipeline import (STRATEGIES, ApeConfig, PrefillOutcome, ape_prefill, cacheblend_prefill, cacheclip_prefill,
                       direct_reuse_prefill, full_attention_prefill, reuse_context_ids)
from .selector import (AuxSelection, ImportanceScores, SelectionConfig, SelectionPlan, WindowRecord,
                       aux_score_tokens, cacheblend_select, map_selection, random_select, select_tokens, selection_budget,
                       top_candidates)
from .tokenizers import AlignmentMap, GreedyTokenizer, TokenSpan, align_spans, char_vocab
from .weights import Model, from_params, init_model, reference_init_params

__version__ = "0.1.0"
