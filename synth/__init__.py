"""Seeded synthetic input generators shared by the tests, smoke() and bench.py.

This package holds NO arithmetic of the method (no softmax, log-prob, advantage,
ratio or gradient): it only draws random inputs with the shapes and structure of the
paper's workloads (DESIGN.md §5 "input recipe").  Both the oracle side and the CUDA
side receive exactly the arrays produced here.  Where an input must be *derived*
from a log-prob (the behaviour log-probs ``old_logp``), the caller passes the
reference log-probs in and this package only adds the seeded perturbation.
"""
from .inputs import *  # noqa: F401,F403
