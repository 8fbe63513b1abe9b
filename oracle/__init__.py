"""Parity oracle (test infrastructure only; see kvpool_oracle.py header)."""
