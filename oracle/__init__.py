"""CPU oracle (test infrastructure only; see dquant_oracle.py header)."""
