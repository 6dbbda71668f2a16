"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see dngd_oracle.py header)."""
