"""Synthetic inputs and the 128-bit result checksum (host-side API objects).

* ``SyntheticSpec`` / ``gen_random_exact`` / ``gen_analytic`` -- verify.py:110-192.
  Runs never call ``local_block`` for these: the engine recognises the spec
  and generates each rank's block directly in HBM (``psim_gen_*``), so the
  generator is not a host bottleneck. ``local_block``
  exists for API compatibility (and is what a host-only consumer would use).
* ``gen_uniform`` -- general-FP inputs from the same hash, for
  tolerance/bitwise tests on non-integer data.
* ``Checksum128`` / ``checksum`` / ``combine_checksums`` -- verify.py:68-103.
  Engine runs compute checksums on the GPU; ``checksum(records)`` is the
  host utility for record lists a caller already holds.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .domain import ConfigError, DataError, dtype_of, field_range, vector_range

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
MIX_C1 = 0xBF58476D1CE4E5B9
MIX_C2 = 0x94D049BB133111EB


def mix64(x: int) -> int:
    """Wrapping 64-bit avalanche mix (verify.py:36-44)."""
    x &= MASK64
    x = ((x ^ (x >> 30)) * MIX_C1) & MASK64
    x = ((x ^ (x >> 27)) * MIX_C2) & MASK64
    return x ^ (x >> 31)


def mix64_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(MIX_C1)
        x ^= x >> np.uint64(27)
        x *= np.uint64(MIX_C2)
        x ^= x >> np.uint64(31)
    return x


def value_bits(value) -> int:
    """Bit pattern of a metric value, FP32 zero-extended (verify.py:58-65)."""
    a = np.asarray(value)
    if a.dtype == np.float32:
        return int(a.view(np.uint32))
    if a.dtype == np.float64:
        return int(a.view(np.uint64))
    raise TypeError(f"metric values must be float32/float64, got {a.dtype}")


@dataclass(frozen=True)
class Checksum128:
    """Order-independent wrapping sum of mix64(index) * (mix64(bits) | 1)."""

    value: int = 0

    def add_term(self, canonical_index: int, bits: int) -> "Checksum128":
        term = mix64(canonical_index) * (mix64(bits) | 1)
        return Checksum128((self.value + term) & MASK128)

    def combine(self, other: "Checksum128") -> "Checksum128":
        return Checksum128((self.value + other.value) & MASK128)

    @classmethod
    def from_words(cls, lo: int, hi: int) -> "Checksum128":
        return cls(((int(hi) & MASK64) << 64) | (int(lo) & MASK64))

    @property
    def hex(self) -> str:
        return format(self.value, "032x")


def checksum(records: Iterable, n_v: int) -> Checksum128:
    """Checksum of a record collection; duplicate tuples raise DataError."""
    seen: set = set()
    total = 0
    for rec in records:
        key = rec.id.indices
        if key in seen:
            raise DataError(f"duplicate result tuple {key}")
        seen.add(key)
        total += mix64(rec.id.canonical_index(n_v)) * (mix64(value_bits(rec.value)) | 1)
    return Checksum128(total & MASK128)


def combine_checksums(parts: Iterable[Checksum128]) -> Checksum128:
    return Checksum128(sum(p.value for p in parts) & MASK128)


# ---------------------------------------------------------------------------
# synthetic sources

KINDS = ("random-exact", "analytic", "uniform")


@dataclass(frozen=True)
class SyntheticSpec:
    """Input defined per global element (q, i).

    random-exact: mix64(seed ^ (q*n_v + i)) mod 2^bits (exact sums, verify.py:126-129)
    analytic:     1 + [q mod n_v == i]                   (closed-form metrics)
    uniform:      (mix64(seed ^ (q*n_v + i)) >> 11) * 2^-53 (FP64), >> 40 * 2^-24 (FP32)
    """

    kind: str
    seed: int
    n_f: int
    n_v: int
    bits: int = 0

    def element(self, q: int, i: int, precision: str = "double"):
        h = mix64(self.seed ^ (q * self.n_v + i))
        if self.kind == "random-exact":
            return h % (1 << self.bits)
        if self.kind == "analytic":
            return 1 + (1 if q % self.n_v == i else 0)
        return (h >> 11) * 2.0**-53 if precision == "double" else (h >> 40) * 2.0**-24

    def check_exactness(self, precision: str) -> None:
        """ConfigError when sums could round (verify.py:149-158)."""
        if self.kind != "random-exact":
            return
        mant = 24 if precision == "single" else 53
        worst = 3 * self.n_f * ((1 << self.bits) - 1)
        if worst >= (1 << mant):
            raise ConfigError(
                f"bits={self.bits} with n_f={self.n_f} overflows exact {precision} "
                f"accumulation (3*n_f*(2^b-1) = {worst} >= 2^{mant})"
            )

    def check_problem(self, problem) -> None:
        if (problem.n_f, problem.n_v) != (self.n_f, self.n_v):
            raise ConfigError(
                f"problem dims ({problem.n_f}, {problem.n_v}) do not match "
                f"synthetic dims ({self.n_f}, {self.n_v})"
            )
        self.check_exactness(problem.precision)

    def local_block(self, problem, grid, coords) -> np.ndarray:
        """Host materialisation (compatibility path; runs generate on device)."""
        self.check_problem(problem)
        f0, f1 = field_range(grid, coords.p_f, self.n_f)
        v0, v1 = vector_range(grid, coords.p_v, self.n_v)
        q = np.arange(f0, f1, dtype=np.uint64)[:, None]
        i = np.arange(v0, v1, dtype=np.uint64)[None, :]
        dt = dtype_of(problem.precision)
        if self.kind == "analytic":
            vals = (q % np.uint64(self.n_v) == i).astype(np.uint64) + np.uint64(1)
            return np.asfortranarray(vals.astype(dt))
        with np.errstate(over="ignore"):
            h = mix64_np((q * np.uint64(self.n_v) + i) ^ np.uint64(self.seed))
        if self.kind == "random-exact":
            return np.asfortranarray((h & np.uint64((1 << self.bits) - 1)).astype(dt))
        if dt == np.float64:
            return np.asfortranarray((h >> np.uint64(11)).astype(np.float64) * 2.0**-53)
        return np.asfortranarray(((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24)))


def gen_random_exact(seed: int, n_f: int, n_v: int, bits: int) -> SyntheticSpec:
    if not 0 <= bits <= 53:
        raise ConfigError(f"magnitude bits must be in [0, 53], got {bits}")
    return SyntheticSpec("random-exact", seed & MASK64, n_f, n_v, bits)


def gen_analytic(seed: int, n_f: int, n_v: int) -> SyntheticSpec:
    if n_f < n_v:
        raise ConfigError(f"analytic input needs n_f >= n_v, got n_f={n_f} n_v={n_v}")
    return SyntheticSpec("analytic", seed & MASK64, n_f, n_v)


def gen_uniform(seed: int, n_f: int, n_v: int) -> SyntheticSpec:
    return SyntheticSpec("uniform", seed & MASK64, n_f, n_v)


def synthetic_kind(source) -> str | None:
    """Kind of a synthetic source (ours or a duck-typed reference spec), else None."""
    kind = getattr(source, "kind", None)
    if kind in KINDS and all(hasattr(source, a) for a in ("seed", "n_f", "n_v")):
        return kind
    return None
