"""CPU oracle (test infrastructure only; see pfr_oracle.py)."""
