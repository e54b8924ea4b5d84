"""Key space, seeded hashing, fingerprints and the table configuration record.

Host-side half of the drop-in boundary.  Everything here is pure integer
arithmetic that must agree bit for bit with the device kernels
(``csrc/ws_device.cuh``) and with the reference package ``warpbench``:

* sentinels            -- reference ``pkg/src/warpbench/core.py:27-31``
* splitmix64 finaliser -- reference ``core.py:120-129``
* seed derivation      -- reference ``core.py:142-148``
* bucket / tag rules   -- reference ``core.py:157-161`` and ``core.py:171-182``
* TableConfig fields   -- reference ``core.py:185-211``
* validation rules     -- reference ``core.py:225-291``
* key=value files      -- reference ``core.py:294-354``

The derived per-design constants the kernels need (seeds, iceberg front
size, shortcut slots, zero-count cap) are computed here in Python, exactly
as the reference computes them, and handed to the C ABI pre-computed; the
device never re-derives a float-dependent quantity.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

U64 = 0xFFFF_FFFF_FFFF_FFFF
MASK64 = U64

# Slot sentinels (reference core.py:27-31).
EMPTY_KEY = 0
TOMBSTONE_KEY = U64
RESERVED_KEY = U64 - 1
SENTINELS = frozenset((EMPTY_KEY, TOMBSTONE_KEY, RESERVED_KEY))

SLOT_BYTES = 16
TAG_BYTES = 2

_PHI64 = 0x9E37_79B9_7F4A_7C15

DESIGNS = ("double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md",
           "cuckoo", "chaining", "unsafe_reference")

# Design-id enumeration shared with include/warpspeed.h (WS_DESIGN_*).
DESIGN_ID = {name: i for i, name in enumerate(DESIGNS)}

# Per-design default bucket sizes (reference core.py:51-61).
DEFAULT_BUCKET_SIZE = dict(zip(DESIGNS, (8, 32, 32, 32, 32, 32, 8, 7, 32)))

MD_DESIGNS = frozenset(("double_md", "p2_md", "iceberg_md"))

# Number of independent hash functions each design consumes
# (reference core.py:66-76).
SEEDS_REQUIRED = dict(zip(DESIGNS, (2, 2, 2, 2, 3, 3, 3, 1, 2)))

MODES = ("concurrent", "phased")
SLOT_ENGINES = ("auto", "wide", "packed")
_PACKED_FROM = 4_000_000   # reference core.py:216


class WarpbenchError(Exception):
    """Root of the library's exception hierarchy."""


class InvalidKeyError(WarpbenchError):
    """A sentinel (or out-of-range integer) was used as a key or value."""


class ConfigError(WarpbenchError):
    """Raised with *all* violated configuration invariants at once."""

    def __init__(self, problems):
        self.problems = list(problems)
        super().__init__("; ".join(self.problems))


def is_sentinel(key: int) -> bool:
    return key in SENTINELS


def check_key(key: int) -> None:
    """Public-boundary key check (reference core.py:107-112)."""
    if key < 0 or key > U64:
        raise InvalidKeyError(f"key {key!r} is outside the unsigned 64-bit range")
    if key in SENTINELS:
        raise InvalidKeyError(f"key {key:#x} is a reserved sentinel")


def check_value(value: int) -> None:
    if value < 0 or value > U64:
        raise InvalidKeyError(f"value {value!r} is outside the unsigned 64-bit range")


def mix64(x: int) -> int:
    """splitmix64 finaliser over 64 bits (same constants as the device)."""
    x &= U64
    x ^= x >> 30
    x = (x * 0xBF58_476D_1CE4_E5B9) & U64
    x ^= x >> 27
    x = (x * 0x94D0_49BB_1331_11EB) & U64
    x ^= x >> 31
    return x


class HashFamily:
    """``count`` seeded functions h_i(k) = mix64(k ^ seed_i)."""

    __slots__ = ("master_seed", "seeds")

    def __init__(self, master_seed: int, count: int = 4):
        if count < 1:
            raise ConfigError(["hash family needs at least one function"])
        self.master_seed = master_seed & U64
        self.seeds = tuple(mix64(self.master_seed + _PHI64 * (i + 1))
                           for i in range(count))

    def __len__(self):
        return len(self.seeds)

    def raw(self, index: int, key: int) -> int:
        return mix64(key ^ self.seeds[index])

    def bucket(self, index: int, key: int, num_buckets: int) -> int:
        # high 48 bits address the bucket, the low 16 feed the tag
        return (self.raw(index, key) >> 16) % num_buckets


def hash_bucket(family: HashFamily, index: int, key: int, num_buckets: int) -> int:
    if num_buckets < 1:
        raise ConfigError(["num_buckets must be >= 1"])
    return family.bucket(index, key, num_buckets)


def fingerprint(family: HashFamily, key: int) -> int:
    """16-bit tag: low half-word of the primary hash, 0 remapped to 1."""
    t = family.raw(0, key) & 0xFFFF
    return t or 1


@dataclass(frozen=True)
class TableConfig:
    """Design selector plus sizing knobs (field names follow the reference)."""

    design: str
    capacity_slots: int
    bucket_size: int = 0
    line_bytes: int = 128
    probe_cap: int = 512
    mode: str = "concurrent"
    seed: int = 0x5EED
    iceberg_front_fraction: float = 0.83
    shortcut_threshold: float = 0.75
    cuckoo_ways: int = 3
    cuckoo_path_depth: int = 5
    slot_engine: str = "auto"

    def hash_family(self) -> HashFamily:
        need = SEEDS_REQUIRED.get(self.design, 3)
        return HashFamily(self.seed, max(need, self.cuckoo_ways, 3))


def resolve_slot_engine(cfg: TableConfig) -> str:
    """Reported engine name.  On the device every slot is one 16-byte cell
    published by a single 128-bit atomic, i.e. always a 'wide' atomic; the
    name is kept for manifest compatibility with the reference."""
    if cfg.slot_engine != "auto":
        return cfg.slot_engine
    return "packed" if cfg.capacity_slots >= _PACKED_FROM else "wide"


def _alignment_problem(cfg: TableConfig, bucket: int):
    if cfg.design == "chaining":
        node = bucket * SLOT_BYTES + 8
        if node > cfg.line_bytes:
            return (f"chaining node ({bucket} pairs + link = {node}B) does not "
                    f"fit one {cfg.line_bytes}B line")
        return None
    span = bucket * SLOT_BYTES
    if span % cfg.line_bytes and 2 * span != cfg.line_bytes:
        return (f"bucket_size {bucket} spans {span}B which is neither a multiple "
                f"nor exactly half of line_bytes {cfg.line_bytes}")
    return None


def validate_config(cfg: TableConfig) -> TableConfig:
    """Fill the default bucket size and check every invariant; raise
    ConfigError naming all violations (reference core.py:225-291)."""
    if cfg.design not in DESIGNS:
        raise ConfigError([f"unknown design {cfg.design!r} (choose from {', '.join(DESIGNS)})"])
    bucket = cfg.bucket_size or DEFAULT_BUCKET_SIZE[cfg.design]
    cfg = dataclasses.replace(cfg, bucket_size=bucket)
    bad = []
    if cfg.mode not in MODES:
        bad.append(f"unknown mode {cfg.mode!r}")
    if cfg.slot_engine not in SLOT_ENGINES:
        bad.append(f"unknown slot_engine {cfg.slot_engine!r}")
    if cfg.line_bytes < SLOT_BYTES or cfg.line_bytes % SLOT_BYTES:
        bad.append(f"line_bytes {cfg.line_bytes} must be a positive multiple of {SLOT_BYTES}")
    if cfg.capacity_slots <= 0:
        bad.append("capacity_slots must be positive")
    if bucket <= 0:
        bad.append("bucket_size must be positive")
    if not bad:
        msg = _alignment_problem(cfg, bucket)
        if msg:
            bad.append(msg)
        if cfg.capacity_slots % bucket:
            bad.append(f"capacity_slots {cfg.capacity_slots} is not a multiple of "
                       f"bucket_size {bucket}")
    if cfg.probe_cap < 1:
        bad.append("probe_cap must be >= 1")
    if not 0.0 < cfg.iceberg_front_fraction < 1.0:
        bad.append("iceberg_front_fraction must be in (0, 1)")
    if not 0.0 <= cfg.shortcut_threshold <= 1.0:
        bad.append("shortcut_threshold must be in [0, 1]")
    if cfg.cuckoo_ways < 2:
        bad.append("cuckoo_ways must be >= 2")
    if cfg.cuckoo_path_depth < 1:
        bad.append("cuckoo_path_depth must be >= 1")
    if cfg.design.startswith("iceberg") and not bad:
        total = cfg.capacity_slots // bucket
        front = round(cfg.capacity_slots * cfg.iceberg_front_fraction / bucket)
        if not 1 <= front <= total - 1:
            bad.append("capacity too small to split into a front yard and a backyard "
                       f"({total} buckets at fraction {cfg.iceberg_front_fraction})")
    if bad:
        raise ConfigError(bad)
    return cfg


# ---------------------------------------------------------------------------
# flat key=value config files (reference core.py:294-354)

_INT_KEYS = frozenset(("capacity_slots", "bucket_size", "line_bytes", "probe_cap",
                       "seed", "cuckoo_ways", "cuckoo_path_depth"))
_FLOAT_KEYS = frozenset(("iceberg_front_fraction", "shortcut_threshold"))


def format_config(cfg: TableConfig) -> str:
    return "".join(f"{f.name}={getattr(cfg, f.name)}\n"
                   for f in dataclasses.fields(TableConfig))


def parse_config(text: str, base: TableConfig | None = None) -> TableConfig:
    names = {f.name for f in dataclasses.fields(TableConfig)}
    got, bad = {}, []
    for n, line in enumerate(text.splitlines(), 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, eq, raw = line.partition("=")
        if not eq:
            bad.append(f"line {n}: expected key=value, got {line!r}")
            continue
        key, raw = key.strip(), raw.strip()
        if key not in names:
            bad.append(f"line {n}: unknown config key {key!r}")
            continue
        try:
            if key in _INT_KEYS:
                got[key] = int(raw, 0)
            elif key in _FLOAT_KEYS:
                got[key] = float(raw)
            else:
                got[key] = raw
        except ValueError:
            bad.append(f"line {n}: bad value {raw!r} for {key}")
    if bad:
        raise ConfigError(bad)
    if base is not None:
        got = {**dataclasses.asdict(base), **got}
    if "design" not in got or "capacity_slots" not in got:
        raise ConfigError(["config must define at least design and capacity_slots"])
    return TableConfig(**got)


def load_config_file(path) -> TableConfig:
    with open(path, encoding="utf-8") as fh:
        return parse_config(fh.read())


# ---------------------------------------------------------------------------
# derived constants handed to the device (never re-derived in C)

@dataclass(frozen=True)
class Derived:
    """Per-table integers the kernels consume, computed the reference's way."""

    design_id: int
    md: bool
    bucket_size: int
    num_buckets: int          # total buckets (slots // bucket)
    primary_buckets: int      # front yard for iceberg, else num_buckets
    front_buckets: int
    back_buckets: int
    seeds: tuple
    shortcut_slots: int       # int(threshold * bs)      -- openaddr.py:351-352
    zero_count_cap: int       # max(1, bs - int(thr*bs) + 1) -- openaddr.py:45-47
    probe_cap: int
    ways: int
    path_depth: int
    phased: bool
    lock_elided: bool


def derive(cfg: TableConfig) -> Derived:
    cfg = validate_config(cfg)
    bs = cfg.bucket_size
    nb = cfg.capacity_slots // bs
    front, back = nb, 0
    if cfg.design.startswith("iceberg"):
        f = round(nb * cfg.iceberg_front_fraction)   # half-even, openaddr.py:505
        front = min(max(f, 1), nb - 1)
        back = nb - front
    sc = int(cfg.shortcut_threshold * bs)
    return Derived(
        design_id=DESIGN_ID[cfg.design],
        md=cfg.design in MD_DESIGNS,
        bucket_size=bs,
        num_buckets=nb,
        primary_buckets=front,
        front_buckets=front,
        back_buckets=back,
        seeds=cfg.hash_family().seeds,
        shortcut_slots=sc,
        zero_count_cap=max(1, bs - sc + 1),
        probe_cap=cfg.probe_cap,
        ways=cfg.cuckoo_ways,
        path_depth=cfg.cuckoo_path_depth,
        phased=cfg.mode == "phased",
        lock_elided=cfg.design == "unsafe_reference",
    )
