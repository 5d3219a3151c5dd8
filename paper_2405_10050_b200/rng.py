"""Deterministic, splittable random streams.

Host-side streams keep the reference contract exactly: ``stream(seed,
purpose, index)`` is ``numpy.random.Generator(PCG64(SeedSequence(entropy=seed,
spawn_key=(tag, index))))`` (pkg/src/voronray/rng.py:10-28), so a descent or
an MC cell driven from a host stream draws bit-identical directions to the
reference.  The device-side MC stream is Philox4x32-10 keyed by the seed with
counter (ray, cell, pair, purpose) -- see csrc/raycast_core.cuh and
:func:`philox_normals_reference_order` for its exact definition.
"""

import numpy as np

PURPOSES = {
    "descent": 0,
    "mc": 1,
    "bench": 2,
    "test": 3,
}


def stream(seed, purpose, index=0):
    """numpy Generator for (seed, purpose, index); same bits as the reference."""
    tag = PURPOSES[purpose]
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(tag, index))
    return np.random.Generator(np.random.PCG64(ss))


class ReplayNormals:
    """Duck-typed ``rng`` that serves pre-drawn standard normals in order.

    ``standard_normal(size)`` returns the next ``prod(size)`` values, which is
    how device Philox directions are replayed into a host consumer that
    expects a numpy Generator (SURVEY.md §8(c) rule 4).
    """

    def __init__(self, values):
        self._v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
        self._pos = 0

    def standard_normal(self, size=None):
        n = 1 if size is None else int(np.prod(size))
        if self._pos + n > self._v.size:
            raise IndexError("replay buffer exhausted")
        out = self._v[self._pos:self._pos + n].copy()
        self._pos += n
        if size is None:
            return float(out[0])
        return out.reshape(size)

    @property
    def remaining(self):
        return self._v.size - self._pos
