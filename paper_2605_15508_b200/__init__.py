"""B200-native (sm_100a) STS sparse-attention hot path.

Drop-in for the hot-path subset of the reference package ``specsparse``
(src/__init__.py:55-102): the sparsity API (SparsityConfig, page_aggregate,
draft_masks_decode, draft_masks_prefill, remap_masks, sparse_attention,
dump_masks), the head-mapping tables (HeadMapping, MappingSet, load/save),
the model-level capture and verify forwards (toymodel's forward_prefill /
forward_decode / forward_block with record_attention / record_scores /
masks: ``model``), the integrated verify loop (specdec's propose / verify /
generate / greedy_generate, device-resident: ``specdec``), the error
classes, and the batched device pipeline (``verify_step.STSVerifyStep``) that
replaces propose -> _verification_masks -> verify for gamma+1 stacked rows.

All compute runs in libsts_b200.so (include/sts_b200.h); there is no CPU
fallback.
"""

from .errors import (
    CapacityError,
    ConfigError,
    ContractViolation,
    DeviceError,
    InputError,
    SpecSparseError,
)
from .headmap import HeadMapping, MappingSet, find_head_mapping, load_mapping, save_mapping
from .model import (ForwardRecord, ModelConfig, PagedKVCache, forward_block, forward_decode, forward_prefill,
                    replay_position)
from .sparsity import (
    SparsityConfig,
    draft_masks_decode,
    draft_masks_prefill,
    dump_masks,
    page_aggregate,
    remap_masks,
    sparse_attention,
    sparse_prefill_attention,
    verification_masks,
)
from .specdec import (GenerateResult, GenerateStats, ModelSession, RoundOutcome, SpecConfig, generate,
                      greedy_generate, propose, verify)

__version__ = "0.1.0"

__all__ = [
    "ForwardRecord",
    "GenerateResult",
    "GenerateStats",
    "ModelConfig",
    "ModelSession",
    "PagedKVCache",
    "RoundOutcome",
    "SpecConfig",
    "forward_block",
    "forward_decode",
    "forward_prefill",
    "generate",
    "greedy_generate",
    "propose",
    "replay_position",
    "save_mapping",
    "verify",
    "CapacityError",
    "ConfigError",
    "ContractViolation",
    "DeviceError",
    "HeadMapping",
    "InputError",
    "MappingSet",
    "SparsityConfig",
    "SpecSparseError",
    "draft_masks_decode",
    "draft_masks_prefill",
    "find_head_mapping",
    "dump_masks",
    "load_mapping",
    "page_aggregate",
    "remap_masks",
    "sparse_attention",
    "sparse_prefill_attention",
    "verification_masks",
]
