"""CPU oracle for parity tests and the CPU baseline — TEST INFRASTRUCTURE ONLY (see mpx_oracle.py)."""
