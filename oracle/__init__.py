"""fp64 CPU oracle for the decomposed-LLM TP hot path (arxiv 2604.17709).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package (``paper_2604_17709_b200``) never imports it,
and this package never imports the product: they share no code.

The arithmetic lives in ``dl_oracle.c`` (plain C, fp64, OpenMP over
independent outputs).  This module only compiles it with gcc and marshals
numpy arrays through ctypes.  See the C file's header for citations.
"""
from .oracle import *  # noqa: F401,F403
