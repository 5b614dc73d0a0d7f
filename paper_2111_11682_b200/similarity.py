"""Neighbour table J^K (reference similarity.py:14-48).

The exact shrunk-Pearson GSM search and the random control of the reference
(similarity.py:51-213) are a quadratic quality oracle and a control, outside
the accelerated path (SURVEY §2 Table A), and are not rebuilt here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class NeighborTable:
    """Per-column Top-K neighbour indices, one row of K entries per column."""

    N: int
    K: int
    entries: np.ndarray  # (N, K) int32

    def validate(self) -> None:
        if self.entries.shape != (self.N, self.K):
            raise ValueError(f"entries shape {self.entries.shape} != ({self.N}, {self.K})")
        e = np.asarray(self.entries)
        if self.K:
            s = np.sort(e, axis=1)
            dup = (s[:, 1:] == s[:, :-1]).any(axis=1) if self.K > 1 else np.zeros(self.N, bool)
            if dup.any():
                raise ValueError(f"duplicate neighbor in row {int(np.flatnonzero(dup)[0])}")
            selfn = (e == np.arange(self.N)[:, None]).any(axis=1)
            if selfn.any():
                raise ValueError(f"self-neighbor in row {int(np.flatnonzero(selfn)[0])}")
            bad = ((e < 0) | (e >= self.N)).any(axis=1)
            if bad.any():
                raise ValueError(f"neighbor index out of range in row {int(np.flatnonzero(bad)[0])}")

    def write_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write("j,rank,neighbor\n")
            for j in range(self.N):
                for rank in range(self.K):
                    fh.write(f"{j},{rank},{self.entries[j, rank]}\n")

    @classmethod
    def read_csv(cls, path) -> "NeighborTable":
        data = np.loadtxt(path, delimiter=",", skiprows=1, dtype=np.int64, ndmin=2)
        N = int(data[:, 0].max()) + 1
        K = int(data[:, 1].max()) + 1
        entries = np.zeros((N, K), dtype=np.int32)
        entries[data[:, 0], data[:, 1]] = data[:, 2]
        return cls(N=N, K=K, entries=entries)
