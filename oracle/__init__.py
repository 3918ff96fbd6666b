"""CPU oracle (test infrastructure only; see shuffle_oracle.py header)."""
