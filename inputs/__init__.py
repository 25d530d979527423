"""Seeded synthetic input generators shared by tests, bench and smoke.

Holds none of the method's arithmetic: only phantom geometry, Gaussian noise
and random states.  Both the oracle and the CUDA path consume its outputs.
"""
from .phantom import *  # noqa: F401,F403
