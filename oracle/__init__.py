"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see tileprep_oracle.py)."""
