"""Philox4x32-10 counter-based random generator, written out in pure Python.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper draws "omega_1, ..., omega_m iid ~ P" (Sec. 2.4
RFDiffusion) but fixes no generator.  The random stream is therefore part of
this build's contract (reading A14): Philox4x32-10 (Salmon et al.,
"Parallel random numbers: as easy as 1, 2, 3", SC'11) with the standard
round constants, ten rounds, and the key bumped between rounds.

Pins: ``tests/test_oracle_philox.py`` checks these words against curand's own
``curand_Philox4x32_10`` compiled for the host (an independent
implementation, used only in that test) and against the published
zero-counter / zero-key known answer 6627e8d5 e169c58d bc57ac4c 9b00dbd8.
"""

MASK32 = 0xFFFFFFFF

# Multipliers and Weyl key increments of Philox4x32 (SC'11, Table 2).
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85


def _mulhilo(a, b):
    """Full 64-bit product of two 32-bit words, split into (hi, lo)."""
    p = a * b
    return (p >> 32) & MASK32, p & MASK32


def _round(ctr, key):
    """One Philox S-box round on a 4-word counter with a 2-word key."""
    hi0, lo0 = _mulhilo(PHILOX_M0, ctr[0])
    hi1, lo1 = _mulhilo(PHILOX_M1, ctr[2])
    return (
        (hi1 ^ ctr[1] ^ key[0]) & MASK32,
        lo1,
        (hi0 ^ ctr[3] ^ key[1]) & MASK32,
        lo0,
    )


def philox4x32_10(counter, key):
    """Philox4x32 with 10 rounds: (4 x u32 counter, 2 x u32 key) -> 4 x u32.

    Round, bump key, round, ..., round: ten rounds, nine key bumps.
    """
    ctr = tuple(int(c) & MASK32 for c in counter)
    k = [int(key[0]) & MASK32, int(key[1]) & MASK32]
    for r in range(10):
        ctr = _round(ctr, k)
        if r != 9:
            k[0] = (k[0] + PHILOX_W0) & MASK32
            k[1] = (k[1] + PHILOX_W1) & MASK32
    return ctr
