"""Seeded, synthetic workload inputs shared by the oracle and the CUDA path.

Holds data and random draws only; none of the method's arithmetic.
"""
