"""CPU oracle -- test infrastructure only (see goat_oracle.py header)."""
