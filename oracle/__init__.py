"""CPU oracle for parity checks -- test infrastructure only (see ogcp_oracle.py)."""
