"""Seeded synthetic inputs shared by the golden generator and the parity tests.

BASELINE.json's configs draw latent weights W ~ N(0, 0.02) in fp32 and
activations x ~ N(0, 1) in fp32; the reference package has no dataset, so the
seeds below *are* the workload.  Host NumPy generation is used for every case
the tests regenerate (PCG64 is platform independent), so a GPU box can rebuild
the exact inputs the golden hashes were taken on without /root/reference.
"""

from __future__ import annotations

import hashlib

import numpy as np


def latent_weights(seed: int, rows: int, cols: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(0.02)


def activations(seed: int, m: int, k: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((m, k), dtype=np.float32)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# Config-shaped parity cases (BASELINE.json configs 0..4).  Each matrix is
# (name, rows N, cols K, weight seed); each activation set is (name, M, K, seed).
LARGE_CASES = {
    "cfg0": {
        "matrices": [("w", 4096, 4096, 0)],
        "acts": [("x", 1, 4096, 1)],
        "gemv": [("w", "x")],
    },
    "cfg1": {
        "matrices": [("gate", 14336, 4096, 10), ("up", 14336, 4096, 11),
                     ("down", 4096, 14336, 12)],
        "acts": [("xh", 1, 4096, 13), ("xi", 1, 14336, 14)],
        "gemv": [("gate", "xh"), ("up", "xh"), ("down", "xi")],
    },
    "cfg2": {
        "matrices": [("q", 4096, 4096, 20), ("k", 1024, 4096, 21),
                     ("v", 1024, 4096, 22), ("o", 4096, 4096, 23),
                     ("gate", 14336, 4096, 24), ("up", 14336, 4096, 25),
                     ("down", 4096, 14336, 26)],
        "acts": [("xh", 1, 4096, 27), ("xi", 1, 14336, 28)],
        "gemv": [("q", "xh"), ("k", "xh"), ("v", "xh"), ("o", "xh"),
                 ("gate", "xh"), ("up", "xh"), ("down", "xi")],
    },
    "cfg3": {  # the whole prefill layer the bench times (q ... down, K up to 14336)
        "matrices": [("q", 4096, 4096, 30), ("k", 1024, 4096, 32), ("v", 1024, 4096, 33),
                     ("o", 4096, 4096, 34), ("gate", 14336, 4096, 35),
                     ("up", 14336, 4096, 36), ("down", 4096, 14336, 37)],
        "acts": [("x", 512, 4096, 31), ("xi", 512, 14336, 38)],
        "gemv": [("q", "x"), ("k", "x"), ("v", "x"), ("o", "x"), ("gate", "x"),
                 ("up", "x"), ("down", "xi")],
    },
    "cfg4": {
        "matrices": [("q", 10240, 10240, 40), ("k", 1280, 10240, 41),
                     ("down", 10240, 32768, 42)],
        "acts": [("xh", 8, 10240, 43), ("xi", 8, 32768, 44)],
        "gemv": [("q", "xh"), ("k", "xh"), ("down", "xi")],
    },
}
