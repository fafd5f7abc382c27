"""B200-native BagPipe embedding-access path with the embcache API.

Drop-in for the reference package's hot path (reference
``pkg/src/embcache/__init__.py:9-100``): the Oracle Cacher planner, the
trainer TTL cache, the embedding server, the stub trainer math and the
pipelined engine / synchronous oracle.  Every per-key operation runs in
hand-written sm_100a CUDA (``csrc/``, exported through the C ABI of
``include/bagpipe_b200.h``); importing the package needs no GPU, calling the
hot path does -- there is no CPU fallback.

Out of scope: skew analytics, the store wire protocol and
the CLI.
"""

from .errors import (
    CacheCapacityError,
    CacheError,
    CacheMissError,
    CacheOrderingError,
    ConfigurationError,
    EmbcacheError,
    EngineError,
    IncomparableRunsError,
    StoreError,
    StoreKeyError,
)
from .report import IterationRecord, RunReport, load_report
from .traces import (
    Batch,
    EmbeddingKey,
    Example,
    Schema,
    ZipfSpec,
    batchify,
    batchify_columns,
    generate_columns,
    generate_synthetic_trace,
    hash_categorical,
    iter_trace,
    parse_criteo_tsv,
    read_trace_columns,
    read_trace_schema,
    write_trace,
)

__version__ = "0.1.0"

_LAZY = {
    "DynamicCache": ".cache",
    "CachePlan": ".lookahead",
    "LookaheadState": ".lookahead",
    "adapt_on_pressure": ".lookahead",
    "auto_lookahead": ".lookahead",
    "emit_next_plan": ".lookahead",
    "format_plan": ".lookahead",
    "new_state": ".lookahead",
    "parse_plan": ".lookahead",
    "plan_trace": ".lookahead",
    "ShardedStore": ".store",
    "initial_values": ".store",
    "StubModelConfig": ".trainer",
    "apply_updates": ".trainer",
    "combine_gradients": ".trainer",
    "local_gradients": ".trainer",
    "split_sync_sets": ".trainer",
    "gradient_core": ".trainer",
    "combine_core": ".trainer",
    "sgd_step": ".trainer",
    "EngineConfig": ".engine",
    "EquivalenceResult": ".engine",
    "run_pipeline": ".engine",
    "run_bagpipe": ".engine",
    "run_synchronous_baseline": ".engine",
    "verify_equivalence": ".engine",
}


def __getattr__(name):
    # torch-backed modules load on first use so `import paper_2202_12429_b200`
    # stays cheap for host-only consumers (trace tooling, report loading).
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    value = getattr(importlib.import_module(mod, __name__), name)
    globals()[name] = value
    return value


__all__ = sorted(set(_LAZY) | {
    "Batch", "CacheCapacityError", "CacheError", "CacheMissError", "CacheOrderingError", "ConfigurationError",
    "EmbcacheError", "EmbeddingKey", "EngineError", "Example", "IncomparableRunsError", "IterationRecord",
    "RunReport", "Schema", "StoreError", "StoreKeyError", "ZipfSpec", "batchify", "batchify_columns",
    "generate_columns", "generate_synthetic_trace", "hash_categorical", "iter_trace", "load_report",
    "parse_criteo_tsv", "read_trace_columns", "read_trace_schema", "write_trace",
})
