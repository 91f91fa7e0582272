"""Host-side tensor-parallel sharding of canonical LUT-GEMM weights.

Pure index bookkeeping (no arithmetic of the method): which rows or columns
of W a rank owns under the two shardings of SURVEY 8(e), and slicing the
canonical planes / alpha / offset accordingly.  Works on numpy arrays or
torch tensors (CPU or CUDA).
"""
from __future__ import annotations


def row_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r*m/P, (r+1)*m/P) -- requires m % P == 0 (equal shards for all-gather)."""
    if m % world:
        raise ValueError(f"m={m} not divisible by world={world}")
    ms = m // world
    return rank * ms, (rank + 1) * ms


def col_range(n: int, g: int, rank: int, world: int) -> tuple[int, int]:
    """Columns [r*n/P, (r+1)*n/P) -- the shard must be whole groups and whole
    32-column words (n/P % g == 0 and % 32 == 0)."""
    if n % world or (n // world) % g or (n // world) % 32:
        raise ValueError(f"n={n} cannot be split into {world} shards of whole g={g} groups")
    ns = n // world
    return rank * ns, (rank + 1) * ns


def shard_rows(planes, alpha, offset, rank: int, world: int):
    """planes [q][m][n/32], alpha [m][G][q], offset [m][G] | None -> this rank's rows."""
    m = planes.shape[1]
    a, b = row_range(m, rank, world)
    return (planes[:, a:b].contiguous() if hasattr(planes, "contiguous") else planes[:, a:b].copy(),
            _c(alpha[a:b]), None if offset is None else _c(offset[a:b]))


def shard_cols(planes, alpha, offset, n: int, g: int, rank: int, world: int):
    """-> this rank's columns: words [c0/32, c1/32), groups [c0/g, c1/g)."""
    c0, c1 = col_range(n, g, rank, world)
    return (_c(planes[:, :, c0 // 32:c1 // 32]), _c(alpha[:, c0 // g:c1 // g]),
            None if offset is None else _c(offset[:, c0 // g:c1 // g]))


def _c(t):
    return t.contiguous() if hasattr(t, "contiguous") else t.copy()
