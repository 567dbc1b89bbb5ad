"""Seeded synthetic workloads (BASELINE.json configs 1-5; DESIGN.md §4 recipe).

The paper evaluates on MNIST with trained weights; neither is in
the container, so every input here is a seeded stand-in with the shape and
value distribution BASELINE.json states.  Nothing in this module performs CKKS
arithmetic; residue draws are plain uniform integers below each prime.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "CFG1", "CFG2_PRIME_BITS", "CFG3", "CFG4", "CFG5B", "ContextConfig",
    "vecmat_inputs", "uniform_residues", "messages", "cnn_weights", "mnist_like_images",
    "deep_chain_plaintexts", "MNIST_MEAN", "MNIST_STD", "CNNWeights",
]

MNIST_MEAN, MNIST_STD = 0.1307, 0.3081   # BASELINE.json config 4


@dataclass(frozen=True)
class ContextConfig:
    """A CKKS parameter set: log2 N, prime bit sizes (specials last), #special, log2 scale, seed."""
    name: str
    logN: int
    bits: tuple
    n_special: int
    scale_log2: int
    seed: int


# config 1: N=8192, [60,40,40,60] last = special, scale 2^40, Philox seed 0
CFG1 = ContextConfig("cfg1-vecmat", 13, (60, 40, 40, 60), 1, 40, 0)
# config 3: N=16384, 8 x 50-bit data + 2 x 50-bit special, scale 2^50, seed 2
CFG3 = ContextConfig("cfg3-keyswitch", 14, (50,) * 10, 2, 50, 2)
# config 4: N=8192, [31, 26 x 6, 31], scale 2^26; seed 3 (not given)
CFG4 = ContextConfig("cfg4-cnn", 13, (31, 26, 26, 26, 26, 26, 26, 31), 1, 26, 3)
# config 5b: N=32768, 20 x 50-bit (18 data + 2 special), scale 2^40, seed 4
CFG5B = ContextConfig("cfg5b-deep-chain", 15, (50,) * 20, 2, 40, 4)


def CFG2_PRIME_BITS(L: int) -> tuple:
    """config 2: ceil(L/2) 60-bit and floor(L/2) 50-bit primes, interleaved from 60."""
    return tuple(60 if i % 2 == 0 else 50 for i in range(L))


def vecmat_inputs(seed: int = 0, n: int = 64, m: int = 10):
    """config 1: x ~ U[-1,1]^n, W ~ N(0, 0.1^2) of shape n x m (in x out)."""
    rng = np.random.default_rng([1, seed])
    x = rng.uniform(-1.0, 1.0, n)
    W = rng.normal(0.0, 0.1, (n, m))
    return x, W


def uniform_residues(primes, N: int, batch: int, seed: int = 1) -> np.ndarray:
    """config 2: residues uniform in [0, q_i); shape [batch][L][N] uint64."""
    rng = np.random.default_rng([2, seed])
    out = np.empty((batch, len(primes), N), dtype=np.uint64)
    for i, q in enumerate(primes):
        out[:, i, :] = rng.integers(0, int(q), size=(batch, N), dtype=np.uint64)
    return out


def messages(count: int, n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Messages z ~ U[lo, hi]^n, one row per ciphertext (config 3/5b)."""
    rng = np.random.default_rng([3, seed])
    return rng.uniform(lo, hi, (count, n))


@dataclass
class CNNWeights:
    """The paper's network: conv 7x7 stride 3, 4 ch -> x^2 -> FC 256->64 -> x^2 -> FC 64->10.
    PyTorch layouts: conv_w [4,1,7,7], fc1_w [64,256], fc2_w [10,64]."""
    conv_w: np.ndarray
    conv_b: np.ndarray
    fc1_w: np.ndarray
    fc1_b: np.ndarray
    fc2_w: np.ndarray
    fc2_b: np.ndarray


def cnn_weights(seed: int = 3) -> CNNWeights:
    """config 4: all weights and biases ~ N(0, 0.1^2)."""
    rng = np.random.default_rng([4, seed])
    return CNNWeights(
        conv_w=rng.normal(0, 0.1, (4, 1, 7, 7)), conv_b=rng.normal(0, 0.1, 4),
        fc1_w=rng.normal(0, 0.1, (64, 256)), fc1_b=rng.normal(0, 0.1, 64),
        fc2_w=rng.normal(0, 0.1, (10, 64)), fc2_b=rng.normal(0, 0.1, 10),
    )


def mnist_like_images(count: int, seed: int = 4, start: int = 0) -> np.ndarray:
    """config 4/5: 28x28 pixels ~ U{0..255}/255, normalised with MNIST mean/std.
    Image i depends only on (seed, i), so shards can be drawn independently."""
    out = np.empty((count, 28, 28), dtype=np.float64)
    for k in range(count):
        rng = np.random.default_rng([5, seed, start + k])
        px = rng.integers(0, 256, (28, 28)).astype(np.float64) / 255.0
        out[k] = (px - MNIST_MEAN) / MNIST_STD
    return out


def deep_chain_plaintexts(count: int, n: int, seed: int = 4) -> np.ndarray:
    """config 5b (A-cfg5b): plaintext slots uniform in {-1/4, +1/4}."""
    rng = np.random.default_rng([6, seed])
    return np.where(rng.integers(0, 2, (count, n)) == 0, -0.25, 0.25)
