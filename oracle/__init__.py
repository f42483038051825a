"""ORACLE TEST INFRASTRUCTURE (CPU checkers) — see oracle/ffi.py. Not product code."""
