"""Counter-based RNG (decomposition independent).

u(seed, n) = 2 * ((splitmix64(seed * 2**40 + n) >> 11) * 2**-53) - 1  in [-1, 1)

n is the GLOBAL x-fastest cell index, so a rank that generates only its
z-slab gets exactly the values the single-GPU run sees (SURVEY.md §8(d),
"RNG").  Seeds: b0 -> 0, noise_t -> 1000 + t, A-epoch e -> 3000 + e,
sphere centres -> 1.
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z):
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed, idx):
    """U[0,1) with 53 random bits, from counter idx (int array)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64(np.uint64(seed) * np.uint64(1 << 40) + idx)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(seed, idx):
    """U[-1,1): 2*uniform01 - 1 (exact in fp64)."""
    return 2.0 * uniform01(seed, idx) - 1.0
