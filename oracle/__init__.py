"""CPU oracle (test infrastructure only; see compressor_oracle.py)."""
