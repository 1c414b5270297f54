"""Parity oracle for the Fier hot path -- test infrastructure only (see oracle.py)."""
