"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NO arithmetic of the method: only model shapes, ranks chosen
from a compression ratio (an input choice), and random tensors.
"""
from .gen import *  # noqa: F401,F403
