"""Pure-Python model of numpy's Philox4x64-10 stream and Generator.integers.

TEST INFRASTRUCTURE ONLY: pins the algorithm the device sampler
(paper_1503_08294_b200/csrc/sample.cu) restates.  numpy is a third-party
dependency of the reference (pkg/pyproject.toml:10, numpy>=1.24; installed
2.3.5); the reference draws its signals with
Generator(Philox(seed)).integers(0, N, size=m) (sampling.py:175-177,
multi.py:151).  This model follows numpy's published algorithm:

* Philox4x64-10 (Random123): 10 rounds of two 64x64->128 multiplies with
  M0 = 0xD2E7470EE14C6C93, M1 = 0xCA5A826395121157 and Weyl key bumps
  W0 = 0x9E3779B97F4A7C15, W1 = 0xBB67AE8584CAA73B; the 256-bit counter is
  incremented BEFORE each block; a block yields four uint64 words, buffered.
* next_uint32 splits a uint64 word: low half first, the high half is kept
  (has_uint32 / uinteger).
* integers(0, N) for N <= 2^32 uses Lemire's bounded method on 32-bit
  draws: m = u32 * N, reject while (m mod 2^32) < (2^32 - N) mod N,
  result m >> 32.  N == 1 returns zeros without drawing.

tests/test_sampler.py checks it against numpy itself (state included).
"""

from __future__ import annotations

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def philox4x64_10(ctr, key):
    c = list(ctr)
    k = list(key)
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK]
        k = [(k[0] + W0) & MASK, (k[1] + W1) & MASK]
    return c


class PhiloxModel:
    def __init__(self, state: dict):
        s = state["state"]
        self.ctr = [int(x) for x in s["counter"]]
        self.key = [int(x) for x in s["key"]]
        self.buf = [int(x) for x in state["buffer"]]
        self.pos = int(state["buffer_pos"])
        self.has = int(state["has_uint32"])
        self.u = int(state["uinteger"])

    def next64(self) -> int:
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & MASK
            if self.ctr[i]:
                break
        self.buf = philox4x64_10(self.ctr, self.key)
        self.pos = 1
        return self.buf[0]

    def next32(self) -> int:
        if self.has:
            self.has = 0
            return self.u
        v = self.next64()
        self.has = 1
        self.u = v >> 32
        return v & 0xFFFFFFFF

    def integers(self, n_excl: int, size: int) -> list[int]:
        if n_excl == 1:
            return [0] * size
        rng = n_excl - 1
        out = []
        for _ in range(size):
            m = self.next32() * n_excl
            left = m & 0xFFFFFFFF
            if left < n_excl:
                thr = (0xFFFFFFFF - rng) % n_excl
                while left < thr:
                    m = self.next32() * n_excl
                    left = m & 0xFFFFFFFF
            out.append(m >> 32)
        return out
