"""Build/run helper for the host-compiled curand Philox known-answer program."""

import os
import shutil
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "kat", "curand_philox_kat.cu")
_BIN = None


def curand_words(pairs):
    """[(counter4, key2)] -> [4-tuple of u32] from curand_Philox4x32_10 (host build)."""
    global _BIN
    if _BIN is None:
        nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        out = os.path.join(tempfile.mkdtemp(prefix="rfd_kat_"), "kat")
        subprocess.run([nvcc, "-Wno-deprecated-gpu-targets", "-o", out, SRC],
                       check=True, capture_output=True)
        _BIN = out
    lines = "".join("%x %x %x %x %x %x\n" % (tuple(c) + tuple(k)) for c, k in pairs)
    res = subprocess.run([_BIN], input=lines, text=True, capture_output=True,
                         check=True)
    return [tuple(int(w, 16) for w in ln.split()) for ln in res.stdout.splitlines()]
