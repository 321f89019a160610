"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no distances, routing, search or merge):
it only draws vectors, label sets and queries (gen.py) and, as fixture tooling, the per-label
graphs that are an *input* to vf_build_index (graphs.py).
"""
