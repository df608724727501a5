"""CPU oracle (test infrastructure only; see spamm_oracle.py header)."""
