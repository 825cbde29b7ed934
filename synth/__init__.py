"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no level DP, no slowdown model, no
scoring, no arg-min).  It only draws profile tables (integer ns), writes them in the
SPEC profile-file format (SPEC.md "External Interfaces" of [MODULE] profiles),
and describes the benchmark configurations of BASELINE.json as plain data.
See DESIGN.md "Input recipe".
"""
from .profiles import (FAMILIES, synthesize_model, lattice_sizes, write_profile_text,
                       Model)
from .configs import (Problem, make_c1, make_c2, make_c3, make_c4, make_c5, make_s6,
                      random_tiny_problem, library_models, qos_3x, c5_problem, problem_hash)

__all__ = ["FAMILIES", "synthesize_model", "lattice_sizes", "write_profile_text", "Model",
           "Problem", "make_c1", "make_c2", "make_c3", "make_c4", "make_c5", "make_s6",
           "random_tiny_problem", "library_models", "qos_3x", "c5_problem", "problem_hash"]
