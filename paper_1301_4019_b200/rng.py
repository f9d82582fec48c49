"""Stream addressing for the GPU resamplers (mirrors pfresample.rng, rng.py:39-74).

A stream is named by (seed, ids).  Its key is two splitmix64-derived words,
``derive_seed(seed, 0, *ids)`` and ``derive_seed(seed, 1, *ids)``; the kernels
never keep generator state, they evaluate a counter-based generator at
(key, element, step), so draws are independent of scheduling and launch
geometry.  Two device generators share the key:

* ``"philox"`` -- Philox4x32-10 over counters (element, step, purpose): the
  fast default;
* ``"numpy"`` -- an exact device replay of numpy's Philox4x64-10 stream as the
  reference consumes it (``RngStream.generator()``), giving bit-identical draws
  to the reference for the same (seed, ids).
"""

from __future__ import annotations

from dataclasses import dataclass, field

_M64 = 0xFFFFFFFFFFFFFFFF
_STEP = 0x9E3779B97F4A7C15


def _avalanche(z: int) -> int:
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(seed: int, *ids: int) -> int:
    """64-bit subseed of (seed, ids): the id count is absorbed first so that
    (s, (2,)) and (s, (2, 0)) never collide (rng.py:39-49)."""
    acc = _avalanche(int(seed))
    words = (len(ids),) + tuple(int(i) for i in ids)
    for v in words:
        acc = _avalanche(acc + _STEP + (v & _M64))
    return acc


@dataclass(frozen=True)
class RngStream:
    """Reproducible random stream addressed by (seed, ids) (rng.py:52-74)."""

    seed: int
    ids: tuple[int, ...] = field(default=())

    def substream(self, *ids: int) -> "RngStream":
        return RngStream(self.seed, self.ids + tuple(int(i) for i in ids))

    def key(self) -> tuple[int, int]:
        """(key0, key1) of the stream: what the kernels are keyed with."""
        return derive_seed(self.seed, 0, *self.ids), derive_seed(self.seed, 1, *self.ids)

    def generator(self):
        """numpy Generator positioned at the start of the stream (host-side
        compatibility helper; the resamplers never call it)."""
        import numpy as np

        k0, k1 = self.key()
        return np.random.Generator(np.random.Philox(key=np.array([k0, k1], dtype=np.uint64)))


def as_stream(rng) -> RngStream:
    if isinstance(rng, RngStream):
        return rng
    if hasattr(rng, "seed") and hasattr(rng, "ids"):  # a pfresample.RngStream works too
        return RngStream(int(rng.seed), tuple(int(i) for i in rng.ids))
    if isinstance(rng, int):
        return RngStream(rng)
    raise TypeError(f"expected an RngStream, got {type(rng).__name__}")
