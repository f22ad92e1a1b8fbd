"""std::mt19937_64 and libstdc++'s std::uniform_real_distribution<double>,
restated so the reference's acceptance suite (proj/tests/acceptance.cpp) can
be replayed draw for draw.

mt19937_64: the standard's parameters ([rand.predef]); seeding per
[rand.eng.mers].  uniform_real_distribution(a, b): a + (b - a) * u with
u = generate_canonical<double, 53> = double(x) / 2^64 for a 64-bit engine
(one draw), clamped below 1 (libstdc++ random.tcc).
"""

_MASK = (1 << 64) - 1


class MT19937_64:
    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self.N
        mt[0] = seed & _MASK
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self.mt, self.idx = mt, self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % self.N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + self.M) % self.N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK


def uniform(rng: MT19937_64, a: float, b: float) -> float:
    u = float(rng()) / 18446744073709551616.0
    if u >= 1.0:
        u = 0.9999999999999999  # nextafter(1, 0)
    return a + (b - a) * u
