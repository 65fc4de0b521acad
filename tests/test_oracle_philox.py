"""Pins for oracle/philox.py (no GPU)."""

import json
import os
import random

from oracle import philox, rfd
from tests._kat import curand_words


def test_zero_counter_zero_key_published_kat():
    # Random123 known-answer vector for philox4x32_10, counter 0, key 0.
    pin = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))[
        "philox4x32_10_zero_kat"]
    assert philox.philox4x32_10(pin["counter"], pin["key"]) == tuple(int(w, 16) for w in pin["words"])


def test_against_curand_host_build():
    rng = random.Random(1234)
    pairs = [((0, 0, 0, 0), (0, 0)),
             ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF))]
    # The exact (counter, key) pairs the frequency stream uses for the five
    # config seeds, first attempts.
    for seed in range(5):
        key = (seed & 0xFFFFFFFF, seed >> 32)
        for k in (0, 1, 15, 255):
            for a in (0, 1):
                pairs.append(((k, a, rfd.FREQ_TAG, 0), key))
    for _ in range(200):
        pairs.append((tuple(rng.getrandbits(32) for _ in range(4)),
                      tuple(rng.getrandbits(32) for _ in range(2))))
    ref = curand_words(pairs)
    got = [philox.philox4x32_10(c, k) for c, k in pairs]
    assert got == ref
