"""Synthetic inputs identical to the reference's generators.

* ``gen_uniform_keys`` / ``derive_seed`` / ``mix64_np`` restate reference
  ``bench/keys.py:18-54`` (numpy PCG64 stream, sentinels rejected) so that the
  GPU and the CPU oracle are fed bit-identical key batches.
* ``zipf_ranks`` is a vectorised rejection-inversion sampler with the same
  envelope as reference ``bench/zipf.py:18-60`` (theta != 1), for batches far
  too large for the per-draw Python generator.  It is seeded with numpy and is
  therefore *not* draw-for-draw identical to ZipfGen; parity never depends on
  that because the same rank array is fed to both sides.
* ``kmer_keys`` builds canonical 31-mer keys (2 bits/base + 1) from a seeded
  synthetic genome for the sharded k-mer-count workload (BASELINE config 5).
"""

from __future__ import annotations

import numpy as np

U64 = (1 << 64) - 1
_RESERVED_FROM = U64 - 1


def mix64_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def gen_uniform_keys(seed: int, count: int) -> np.ndarray:
    """``count`` uniform non-sentinel uint64 keys from PCG64(seed)."""
    gen = np.random.default_rng(seed & U64)
    out = np.empty(count, dtype=np.uint64)
    have = 0
    while have < count:
        draw = gen.integers(0, 2**64, size=count - have, dtype=np.uint64)
        draw = draw[(draw != 0) & (draw < np.uint64(_RESERVED_FROM))]
        out[have:have + draw.size] = draw
        have += draw.size
    return out


def gen_uniform_key_list(seed: int, count: int) -> list:
    """The same stream as gen_uniform_keys as plain ints, for scalar table
    calls (reference bench/keys.py:43-45)."""
    return gen_uniform_keys(seed, count).tolist()


def derive_seed(master: int, *parts: int) -> int:
    x = master & U64
    for p in parts:
        x = (x * 0x9E3779B97F4A7C15 + p + 1) & U64
        x ^= x >> 29
    return x


def zipf_ranks(n: int, count: int, theta: float = 0.99, seed: int = 0) -> np.ndarray:
    """Ranks in [1, n] with P(k) ~ k^-theta, by vectorised rejection inversion."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if theta < 0 or theta == 1.0:
        raise ValueError("theta must be >= 0 and != 1")
    q = 1.0 - theta

    def hint(x):
        return (np.exp(q * np.log(x)) - 1.0) / q

    def hinv(u):
        return np.exp(np.log1p(u * q) / q)

    h_x1 = hint(np.float64(1.5)) - 1.0
    h_n = hint(np.float64(n + 0.5))
    s = 2.0 - hinv(hint(np.float64(2.5)) - 2.0 ** -theta)
    rng = np.random.default_rng(derive_seed(seed, n, int(theta * 1e6)))
    out = np.empty(count, dtype=np.int64)
    todo = np.arange(count)
    while todo.size:
        u = h_n + rng.random(todo.size) * (h_x1 - h_n)
        x = hinv(u)
        k = np.clip(np.floor(x + 0.5), 1, n)
        ok = (k - x <= s) | (u >= hint(k + 0.5) - np.exp(-theta * np.log(k)))
        out[todo[ok]] = k[ok].astype(np.int64)
        todo = todo[~ok]
    return out


_BASE2 = np.array([0, 1, 2, 3], dtype=np.uint64)


def kmer_keys(genome_len: int, k: int = 31, seed: int = 0, repeats: int = 1) -> np.ndarray:
    """Canonical k-mers of a seeded synthetic genome, packed 2 bits/base, +1.

    The genome is `repeats` back-to-back copies of a random base sequence, so
    every k-mer of the base occurs ~`repeats` times (known multiplicities).
    The +1 keeps every key clear of EMPTY_KEY (reference apps/tensor.py:119);
    k <= 31 keeps it below the RESERVED/TOMBSTONE sentinels.
    """
    if not 1 <= k <= 31:
        raise ValueError("k must be in [1, 31]")
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 4, size=max(k, genome_len // max(1, repeats)), dtype=np.uint64)
    bases = np.tile(base, max(1, repeats))[:genome_len]
    n = genome_len - k + 1
    fwd = np.zeros(n, dtype=np.uint64)
    rev = np.zeros(n, dtype=np.uint64)
    comp = np.uint64(3) - bases
    for i in range(k):
        fwd = (fwd << np.uint64(2)) | bases[i:i + n]
        rev = rev | (comp[i:i + n] << np.uint64(2 * i))
    return np.minimum(fwd, rev) + np.uint64(1)
