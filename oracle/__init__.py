"""CPU oracle (test infrastructure only; see sts_oracle.py header)."""
