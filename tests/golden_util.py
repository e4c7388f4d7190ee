"""Helpers shared by the tests that read the headline-size fixtures."""
import numpy as np

HASH_P = np.uint64(0x100000001B3)


def ext_checksums(ext):
    """Per path: sum_i bits(ext.flat[i]) * P^(i+1) mod 2^64 over the row-major
    ext[rows][cols] -- the checksum oracle/make_golden_big.py stores."""
    n = ext.shape[0]
    bits = np.ascontiguousarray(ext).reshape(n, -1).view(np.uint64)
    w = np.empty(bits.shape[1], dtype=np.uint64)
    acc = np.uint64(1)
    with np.errstate(over="ignore"):
        for i in range(bits.shape[1]):
            acc = acc * HASH_P
            w[i] = acc
        return (bits * w[None, :]).sum(axis=1, dtype=np.uint64)
