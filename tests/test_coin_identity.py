"""The sampler decides a coin on one 32-bit word (sampler.cu coin_zhi): with z the splitmix64
value before its last step x = z ^ (z >> 31) (rng.hpp:15-20), and T' = T << 11 the shifted
threshold (x >> 11 < T  <=>  x < T'), the device uses

    x < T'  ==  hi(z) < hi(T')        whenever hi(z) ^ hi(T') > 1,

and resolves the remaining window exactly.  This checks the identity on random and edge
words (CPU, no device)."""
import numpy as np

M64 = (1 << 64) - 1
EDGE = [0, 1, 2, 3, 0x7FFFFFFE, 0x7FFFFFFF, 0x80000000, 0x80000001, 0x80000002, 0xFFFFFFFE, 0xFFFFFFFF]


def _holds(zhi, zlo, thi, tlo):
    z = (zhi << 32) | zlo
    x = z ^ (z >> 31)
    t = (thi << 32) | tlo
    return (zhi ^ thi) <= 1 or ((x < t) == (zhi < thi))


def test_identity_edge_words():
    for zhi in EDGE:
        for thi in EDGE:
            for zlo in (0, 1, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFF):
                for tlo in (0, 1, 0x80000000, 0xFFFFFFFF):
                    assert _holds(zhi, zlo, thi, tlo), (zhi, zlo, thi, tlo)


def test_identity_random_words():
    rng = np.random.default_rng(5)
    zhi = rng.integers(0, 1 << 32, 200_000, dtype=np.uint64)
    # thresholds near zhi (the interesting region) and anywhere
    near = zhi ^ rng.integers(0, 8, zhi.size, dtype=np.uint64)
    far = rng.integers(0, 1 << 32, zhi.size, dtype=np.uint64)
    thi = np.where(rng.random(zhi.size) < 0.5, near, far)
    zlo = rng.integers(0, 1 << 32, zhi.size, dtype=np.uint64)
    tlo = rng.integers(0, 1 << 32, zhi.size, dtype=np.uint64)
    z = (zhi << np.uint64(32)) | zlo
    x = z ^ (z >> np.uint64(31))
    t = (thi << np.uint64(32)) | tlo
    outside = (zhi ^ thi) > 1
    assert np.array_equal((x < t)[outside], (zhi < thi)[outside])
