"""Independent numpy re-implementation of the SURVEY §8(d) input generator.

Used only to cross-check the two generators (oracle C and CUDA); it holds none
of the method's arithmetic."""
import numpy as np

M64 = (1 << 64) - 1


def splitmix64_np(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_np(seed: int, T: int, D: int, row0: int = 0) -> np.ndarray:
    idx = np.arange(row0 * D, (row0 + T) * D, dtype=np.uint64)
    k = (splitmix64_np(seed, idx) >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (k.astype(np.float32) * np.float32(2.0 ** -23)).reshape(T, D)


def splitmix64_py(seed: int, i: int) -> int:
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def outlier_np(seed: int, T: int, D: int, row0: int = 0) -> np.ndarray:
    """dist 1: column d of the uniform lattice scaled by 2^e_d,
    e_d = (splitmix64(seed ^ 0xC0FFEE, d) mod 9) - 4 (exact: powers of two)."""
    e = (splitmix64_np(seed ^ 0xC0FFEE, np.arange(D, dtype=np.uint64)) % np.uint64(9)).astype(np.int64) - 4
    return (uniform_np(seed, T, D, row0) * np.exp2(e).astype(np.float32)).astype(np.float32)


def ongrid_np(seed: int, T: int, D: int, row0: int = 0) -> np.ndarray:
    """dist 2: x = c * s_d, s_d = j_d 2^-24 with j_d = (splitmix64(seed ^ 0x5CA1E, d) >> 47) | 1,
    c = splitmix64(seed, t D + d) mod 255 - 127, and row 0 forced to +-127 by bit 0 of splitmix64(seed ^ 0x516E, d)."""
    d = np.arange(D, dtype=np.uint64)
    j = (splitmix64_np(seed ^ 0x5CA1E, d) >> np.uint64(47)) | np.uint64(1)
    s = j.astype(np.float32) * np.float32(2.0 ** -24)
    idx = np.arange(row0 * D, (row0 + T) * D, dtype=np.uint64)
    c = (splitmix64_np(seed, idx) % np.uint64(255)).astype(np.int64).reshape(T, D) - 127
    if row0 == 0 and T > 0:
        c[0] = np.where(splitmix64_np(seed ^ 0x516E, d) & np.uint64(1), 127, -127)
    return (c.astype(np.float32) * s).astype(np.float32)
