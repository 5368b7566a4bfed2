"""Philox4x32-10 (Random123) — oracle's own implementation, test infrastructure only.

Used for the seeded draws the method makes (readings R17, R20): the initial
point (counter (r, var, 0, tag 0|1)) and randomised rounding R(a) (counter
(r, var, stage, tag 2)); key = (seed & 0xffffffff, seed >> 32).
Round:  (c0,c1,c2,c3) <- (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0));
        k0 += W0, k1 += W1.
"""
from __future__ import annotations

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (int(x) & MASK for x in ctr)
    k0, k1 = (int(x) & MASK for x in key)
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c3 ^ k1) & MASK, p0 & MASK
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    return c0, c1, c2, c3


def key_of(seed: int):
    return seed & MASK, (seed >> 32) & MASK


def draw24(seed: int, restart: int, var: int, stage: int, tag: int) -> int:
    """24-bit draw k = out0 >> 8 at counter (restart, var, stage, tag)."""
    return philox4x32_10((restart, var, stage, tag), key_of(seed))[0] >> 8


TAG_INIT_A = 0
TAG_INIT_B = 1
TAG_ROUND = 2
