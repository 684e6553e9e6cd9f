"""CPU oracle for the OPC front-end -- test infrastructure only (see flatpoly_oracle.py)."""
