"""Shared helpers of the GPU parity tests (input recipes + boundary query sets)."""
import numpy as np

B, S = 496, 128 * 496          # BiRank16
B4, S4 = 224, 256 * 224        # QuadRank16 (reading R5)


def boundary_queries(n: int, block: int, sblock: int, anchor: int, limit: int = 20000) -> np.ndarray:
    """{0, 1, n-1, n} and every block / anchor / superblock boundary +-1 (capped), within [0, n]."""
    qs = {0, 1, max(n - 1, 0), n}
    for base in range(0, n + 1, block):
        for d in (-1, 0, 1):
            qs.add(base + d)
            qs.add(base + anchor + d)
        if len(qs) > limit:
            break
    for base in range(0, n + 1, sblock):
        for d in (-1, 0, 1):
            qs.add(base + d)
    return np.array(sorted(x for x in qs if 0 <= x <= n), dtype=np.uint64)


def to_dev(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def to_host(t) -> np.ndarray:
    return t.cpu().numpy()
