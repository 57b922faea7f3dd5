"""Synthetic inputs: hierarchical Philox streams and Brownian random walks.

Restates the reference's input generator bit for bit (rng.py:19-70,
sequences.py:34-66 and 110-137) so benchmark and test inputs are identical
to the reference's without importing it. Host-side numpy: inputs only, not
part of the compute path.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["SeedStream", "SequenceBatch", "gen_brownian"]


def _label_words(label: str) -> tuple[int, int]:
    digest = hashlib.blake2b(label.encode("utf-8"), digest_size=8).digest()
    value = int.from_bytes(digest, "little")
    return value & 0xFFFFFFFF, value >> 32


class SeedStream:
    """Root seed plus a label path; immutable (rng.py:26-70)."""

    __slots__ = ("seed", "path", "_key")

    def __init__(self, seed: int, path: tuple = ()):
        if not isinstance(seed, (int, np.integer)) or isinstance(seed, bool):
            raise ValueError(f"seed must be an integer, got {seed!r}")
        if seed < 0 or seed > 0xFFFFFFFFFFFFFFFF:
            raise ValueError(f"seed must fit in an unsigned 64-bit integer, got {seed}")
        self.seed = int(seed)
        self.path = tuple(path)
        key: list[int] = []
        for label in self.path:
            key.extend(_label_words(label))
        self._key = tuple(key)

    def child(self, label: str) -> "SeedStream":
        if not isinstance(label, str) or not label:
            raise ValueError(f"child label must be a non-empty string, got {label!r}")
        return SeedStream(self.seed, self.path + (label,))

    def generator(self) -> np.random.Generator:
        seq = np.random.SeedSequence(entropy=self.seed, spawn_key=self._key)
        return np.random.Generator(np.random.Philox(seq))

    def __eq__(self, other) -> bool:
        return isinstance(other, SeedStream) and (self.seed, self.path) == (other.seed, other.path)

    def __hash__(self) -> int:
        return hash((self.seed, self.path))

    def __repr__(self) -> str:
        return f"SeedStream(seed={self.seed}, path={self.path!r})"


@dataclass
class SequenceBatch:
    """N sequences of L points in R^d as one (N, L, d) float64 array."""

    data: np.ndarray
    ids: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim != 3:
            raise ValueError(f"batch data must be (N, L, d), got shape {self.data.shape}")
        if self.ids is None:
            self.ids = np.arange(self.data.shape[0], dtype=np.int64)

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def length(self) -> int:
        return self.data.shape[1]

    @property
    def dim(self) -> int:
        return self.data.shape[2]


def gen_brownian(n: int, length: int, dim: int, seed: SeedStream, drift=None,
                 start: int = 0) -> SequenceBatch:
    """Brownian walks from the origin with N(0, 1/(length-1)) steps (sequences.py:110-137).

    Sequence k draws from child stream `seq{start + k}`, so any window of a
    batch equals the same rows of the full batch (prefix/window stable).
    """
    if n < 1:
        raise ValueError(f"need n >= 1 sequences, got {n}")
    if length < 2:
        raise ValueError(f"need length >= 2 points, got {length}")
    if dim < 1:
        raise ValueError(f"need dim >= 1 channels, got {dim}")
    drift_vec = np.zeros(dim) if drift is None else np.broadcast_to(
        np.asarray(drift, dtype=np.float64), (dim,))
    scale = math.sqrt(1.0 / (length - 1))
    data = np.empty((n, length, dim))
    data[:, 0, :] = 0.0
    for k in range(n):
        rng = seed.child(f"seq{start + k}").generator()
        steps = rng.standard_normal((length - 1, dim)) * scale + drift_vec
        np.cumsum(steps, axis=0, out=data[k, 1:, :])
    return SequenceBatch(data)
