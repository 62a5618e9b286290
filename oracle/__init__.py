"""CPU oracle package -- test infrastructure only (see srp_oracle.py header)."""
