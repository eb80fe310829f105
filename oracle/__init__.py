"""CPU oracle (test infrastructure only; see burst_oracle.py header)."""
