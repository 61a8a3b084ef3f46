"""Seeded synthetic inputs shared by the golden generator and the tests.

Fixtures store a checksum of each regenerated input rather than the input, which
keeps ``tests/golden`` small. numpy's PCG64 stream and ``standard_normal`` are
identical in this container and on the GPU box, because both run the same image.
"""

import hashlib

import numpy as np


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def spiked(seed: int, p: int, n: int, lams) -> np.ndarray:
    """(p, n) float32: U diag(sqrt(lams)) z + N(0, I), U a seeded orthonormal basis."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((p, len(lams))))
    z = rng.standard_normal((len(lams), n))
    return (U @ (np.sqrt(np.asarray(lams, dtype=np.float64))[:, None] * z) + rng.standard_normal((p, n))).astype(
        np.float32
    )


def mixture(seed: int, p: int, n: int, K: int, scale: float) -> np.ndarray:
    """(p, n) float32 Gaussian mixture: centers scale*N(0, I), unit noise, uniform labels."""
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((p, K)) * scale
    lab = rng.integers(0, K, n)
    return (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
