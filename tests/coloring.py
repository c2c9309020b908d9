"""Test-side graph colouring (host logic, independent of the library): greedy colouring of the
symmetrised sparsity pattern in natural row order, smallest colour not used by an already coloured
neighbour.  Used to give the GPU and the oracle the SAME multicolour SSOR order."""
import numpy as np


def greedy_colors(n, row_ptr, col_idx):
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int64)
    rows = np.repeat(np.arange(n), np.diff(rp))
    # symmetrised adjacency as CSR of (rows, ci) + (ci, rows)
    a = np.concatenate([rows, ci])
    b = np.concatenate([ci, rows])
    keep = a != b
    a, b = a[keep], b[keep]
    order = np.lexsort((b, a))
    a, b = a[order], b[order]
    ptr = np.searchsorted(a, np.arange(n + 1))
    col = -np.ones(n, dtype=np.int64)
    for r in range(n):
        nb = b[ptr[r]:ptr[r + 1]]
        used = set(col[nb[col[nb] >= 0]].tolist())
        c = 0
        while c in used:
            c += 1
        col[r] = c
    return col.astype(np.int32)


def is_valid(n, row_ptr, col_idx, colors):
    rp = np.asarray(row_ptr)
    rows = np.repeat(np.arange(n), np.diff(rp))
    ci = np.asarray(col_idx)
    off = rows != ci
    return not np.any(colors[rows[off]] == colors[ci[off]])
