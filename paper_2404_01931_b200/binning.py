"""Space hash view (flipsim/binning.py:15-24).

offset/count are int32 in HBM (N < 2^31 per device) and widened to int64
on download so the accessor types match the reference.
"""

from __future__ import annotations

import numpy as np


class SpaceHash:
    """Per-cell [offset, offset+count) segments into the cell-sorted particles."""

    def __init__(self, device=None, offset=None, count=None, fluid_cells=None):
        self._dev = device
        if device is None:
            self._offset = np.asarray(offset, dtype=np.int64)
            self._count = np.asarray(count, dtype=np.int64)
            self._fluid = (np.flatnonzero(self._count > 0).astype(np.int64)
                           if fluid_cells is None else np.asarray(fluid_cells, dtype=np.int64))

    @property
    def offset(self) -> np.ndarray:
        return self._dev.hash_arrays()[0] if self._dev is not None else self._offset

    @property
    def count(self) -> np.ndarray:
        return self._dev.hash_arrays()[1] if self._dev is not None else self._count

    @property
    def fluid_cells(self) -> np.ndarray:
        """Ascending raw indices of cells holding particles (binning.py:95)."""
        return self._dev.fluid_cells() if self._dev is not None else self._fluid

    def segment(self, cell: int) -> slice:
        start = int(self.offset[cell])
        return slice(start, start + int(self.count[cell]))
