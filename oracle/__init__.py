"""Test-only CPU oracles (see oracle.py)."""
