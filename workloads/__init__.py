"""Seeded synthetic inputs (graphs, int64 C/M, fractional S*, thresholds, budgets).

Shared by the oracle tests and the CUDA path; holds none of the method's
arithmetic (SURVEY §8(d) input recipe)."""
