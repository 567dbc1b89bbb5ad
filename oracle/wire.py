"""Reference packer of the ciphertext wire format — TEST INFRASTRUCTURE ONLY.

Format (DESIGN.md §3 "wire format", "427KB of communication"):
a 64-byte header followed by, for every item b, poly p, limb i (in that order), the N stored
NTT-domain words of limb i, each written with w_i = bit_length(q_i) bits, least significant bit
first, into a little-endian stream of 64-bit words.  N * w_i is a multiple of 64 for N >= 64, so
every limb segment starts on a 64-bit boundary.  Header (little-endian):
  magic b"HECKKS01" | u32 log2N | u32 B | u32 size | u32 level | f64 scale | u64 payload_bytes
  | u32 n_limbs | 20 zero bytes
Written here with plain Python integers from that definition.
"""
from __future__ import annotations

import struct

import numpy as np

HEADER_BYTES = 64
MAGIC = b"HECKKS01"
MAGIC_SEEDED = b"HECKKSS1"


def limb_widths(primes, level: int) -> list:
    return [int(q).bit_length() for q in primes[: level + 1]]


def payload_bytes(N: int, B: int, size: int, widths) -> int:
    return B * size * N * sum(widths) // 8


def pack(words: np.ndarray, primes, level: int, scale: float) -> bytes:
    """words: [B][size][level+1][N] uint64 -> bytes."""
    B, size, nl, N = words.shape
    assert nl == level + 1
    widths = limb_widths(primes, level)
    out = bytearray()
    for b in range(B):
        for p in range(size):
            for i in range(nl):
                w = widths[i]
                acc, nbits = 0, 0
                seg = bytearray()
                for x in words[b, p, i]:
                    acc |= int(x) << nbits
                    nbits += w
                    while nbits >= 64:
                        seg += (acc & ((1 << 64) - 1)).to_bytes(8, "little")
                        acc >>= 64
                        nbits -= 64
                assert nbits == 0
                out += seg
    hdr = MAGIC + struct.pack("<IIIIdQI", N.bit_length() - 1, B, size, level, float(scale), len(out), nl)
    hdr += bytes(HEADER_BYTES - len(hdr))
    return bytes(hdr) + bytes(out)


def pack_seeded(c0_words: np.ndarray, primes, level: int, scale: float, a_seed: int, stream0: int) -> bytes:
    """Seeded form of a fresh symmetric ciphertext: c0_words [B][level+1][N]; header
    magic b"HECKKSS1", size field 2, the 20-byte tail = u64 a_seed | u64 stream0 | 4 zero bytes;
    payload = the c0 limbs packed exactly as pack() packs a size-1 batch."""
    B = c0_words.shape[0]
    body = pack(c0_words.reshape(B, 1, level + 1, -1), primes, level, scale)[HEADER_BYTES:]
    N = c0_words.shape[-1]
    hdr = MAGIC_SEEDED + struct.pack("<IIIIdQIQQ", N.bit_length() - 1, B, 2, level, float(scale), len(body),
                                     level + 1, a_seed, stream0)
    hdr += bytes(HEADER_BYTES - len(hdr))
    return bytes(hdr) + body
