"""Synthetic test matrices shared by the CPU and GPU tests."""
import numpy as np

import oracle_ref as O


def long_row_csr(n=3000, long_rows=(2999, 2500), width=1200, seed=11):
    """Diagonally dominant CSR with a few rows far longer than a task-level
    plan's per-task buffers (512 entries): chains are cut there and the
    oversize tasks run on the thread-per-task kernel."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        cols = set(rng.choice(n, size=6, replace=False).tolist()) | {i, max(i - 1, 0)}
        if i in long_rows:
            cols |= set(range(max(0, i - width), i))
        rows.append(sorted(cols))
    rp = np.zeros(n + 1, np.int64)
    for i, c in enumerate(rows):
        rp[i + 1] = rp[i] + len(c)
    cols = np.concatenate([np.asarray(c, np.int32) for c in rows])
    vals = rng.uniform(-1.0, 1.0, len(cols)) * 1e-3
    for i in range(n):
        d = rp[i] + rows[i].index(i)
        vals[d] = 4.0 + i % 7
    return O.Csr(rp, cols, vals)
