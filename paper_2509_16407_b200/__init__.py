"""B200-native (sm_100a) WarpSpeed concurrent hash tables.

Drop-in for the reference package ``warpbench``'s table API
(``make_table(TableConfig)`` -> ``HashTable.upsert / query / erase`` plus
introspection), backed by hand-written CUDA kernels behind the C ABI in
``include/warpspeed.h``.  Batched ops take torch tensors and run on the
current CUDA stream.  ``paper_2509_16407_b200.sharded`` spreads one table
over several GPUs (one process per GPU, NCCL all-to-all routing).
"""

from .core import (
    DESIGNS,
    EMPTY_KEY,
    RESERVED_KEY,
    TOMBSTONE_KEY,
    ConfigError,
    HashFamily,
    InvalidKeyError,
    TableConfig,
    WarpbenchError,
    fingerprint,
    format_config,
    parse_config,
    validate_config,
)

__version__ = "0.1.0"


def __getattr__(name):
    # tables import torch lazily so config / hashing work without it
    if name in ("HashTable", "UpsertStatus", "make_table", "merge_id"):
        from . import tables
        return getattr(tables, name)
    raise AttributeError(name)


__all__ = ["DESIGNS", "EMPTY_KEY", "RESERVED_KEY", "TOMBSTONE_KEY", "ConfigError", "HashFamily",
           "InvalidKeyError", "TableConfig", "WarpbenchError", "fingerprint", "format_config",
           "parse_config", "validate_config", "HashTable", "UpsertStatus", "make_table",
           "merge_id", "__version__"]
