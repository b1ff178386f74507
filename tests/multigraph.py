"""Seeded small multigraphs for the symmetry-validator tests (CPU emulation and GPU)."""

import numpy as np


def csr_multi(n, keys):
    """CSR from (src << 32 | dst) keys keeping multiplicities (rows sorted)."""
    keys = np.sort(np.asarray(keys, dtype=np.uint64))
    src = (keys >> np.uint64(32)).astype(np.int64)
    tgt = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))]).astype(np.int64)
    return off, tgt


def perturbed(rng, trial):
    """Skewed symmetric multigraph (hubs at small ids, self-loops, parallel copies), then by
    trial % 4: unchanged, one slot dropped, one slot added, or one slot retargeted."""
    n = int(rng.integers(2, 80))
    m = int(rng.integers(1, 4 * n))
    s = (rng.random(m) ** 3 * n).astype(np.int64)
    d = rng.integers(0, n, m)
    keys = np.concatenate([(s << 32) | d, (d << 32) | s]).astype(np.uint64)
    if trial % 5 == 1:
        keys = np.concatenate([keys, keys[rng.integers(0, keys.shape[0], 3)]])
    op = trial % 4
    if op == 1:
        keys = np.delete(keys, int(rng.integers(0, keys.shape[0])))
    elif op == 2:
        keys = np.append(keys, np.uint64((int(rng.integers(0, n)) << 32) | int(rng.integers(0, n))))
    elif op == 3:
        i = int(rng.integers(0, keys.shape[0]))
        keys[i] = (keys[i] & ~np.uint64(0xFFFFFFFF)) | np.uint64(int(rng.integers(0, n)))
    return (n,) + csr_multi(n, keys)
