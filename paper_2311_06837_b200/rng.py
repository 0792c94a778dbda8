"""Host-side keyed SplitMix64 helpers (rng.hpp:11-61) for seed derivation.
Bulk draws run on the device (gdx_init_uniform); these are scalar conveniences."""

_M = (1 << 64) - 1
_G = 0x9e3779b97f4a7c15


def _fin(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & _M
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & _M
    return z ^ (z >> 31)


def mix64(x: int) -> int:
    """rng.hpp:11-16."""
    return _fin((x + _G) & _M)


class KeyedRng:
    """rng.hpp:18-52."""

    def __init__(self, seed: int, k1: int = 0, k2: int = 0):
        s = mix64(seed & _M)
        s = mix64(s ^ ((k1 + _G) & _M))
        self.state = mix64(s ^ ((k2 + 0xc2b2ae3d27d4eb4f) & _M))

    def next_u64(self) -> int:
        self.state = (self.state + _G) & _M
        return _fin(self.state)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        return (self.next_u64() * n) >> 64

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()
