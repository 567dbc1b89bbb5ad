"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds none of the method's arithmetic: only input draws (messages, images,
weights, residues) with the shapes and distributions of BASELINE.json's configs.
"""
from .inputs import *  # noqa: F401,F403
