"""Philox4x32-10 restated in numpy -- TEST INFRASTRUCTURE for the opt-in
counter-based generator (stk_set_rng(STK_RNG_PHILOX)).  The algorithm is the
published one (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
as 1, 2, 3", SC'11; the generator behind cuRAND's Philox4_32_10 and
Random123): 10 rounds of (hi, lo) = 0xD2511F53 * c0, 0xCD9E8D57 * c2;
c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key += (0x9E3779B9, 0xBB67AE85).
Pinned by the Random123 known-answer vectors (KAT below)."""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)

# (counter, key) -> output, Random123 kat_vectors "philox4x32 10"
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def philox4x32_10(ctr, key):
    """ctr: (..., 4) uint32, key: (..., 2) uint32 -> (..., 4) uint32."""
    c = [np.asarray(ctr, np.uint32)[..., i].astype(np.uint64) for i in range(4)]
    k0 = np.asarray(key, np.uint32)[..., 0].copy()
    k1 = np.asarray(key, np.uint32)[..., 1].copy()
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ k0.astype(np.uint64), lo1, hi0 ^ c[3] ^ k1.astype(np.uint64), lo0]
        with np.errstate(over="ignore"):
            k0 = (k0 + W0).astype(np.uint32)
            k1 = (k1 + W1).astype(np.uint32)
    return np.stack([x.astype(np.uint32) for x in c], axis=-1)


def u64x2(seed, k, j):
    """The device's philox_u64x2: block (k, j) of key = seed -> two u64 words."""
    k = np.asarray(k, np.uint64)
    ctr = np.stack([(k & MASK).astype(np.uint32), (k >> np.uint64(32)).astype(np.uint32),
                    np.full(k.shape, j, np.uint32), np.zeros(k.shape, np.uint32)], axis=-1)
    key = np.broadcast_to(np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32), ctr.shape[:-1] + (2,))
    v = philox4x32_10(ctr, key).astype(np.uint64)
    return (v[..., 0] << np.uint64(32)) | v[..., 1], (v[..., 2] << np.uint64(32)) | v[..., 3]


def csr_rect(n, xmin, xmax, ymin, ymax, p0, p1, seed):
    """The device's Philox CSR on a rectangle (attempt 0 always accepted)."""
    k = np.arange(n, dtype=np.uint64)
    ux, uy = u64x2(seed, k, 0)
    ut, _ = u64x2(seed, k, 1)
    r01 = lambda u: (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    x = xmin + (xmax - xmin) * r01(ux)
    y = ymin + (ymax - ymin) * r01(uy)
    ntl = p1 - p0 + 1
    t = np.array([p0 + ((int(u) * ntl) >> 64) for u in ut], np.int64)
    return x, y, t
