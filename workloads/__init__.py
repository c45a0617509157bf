"""Benchmark / test workload inputs (see meshes.py)."""
