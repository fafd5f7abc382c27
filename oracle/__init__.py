"""CPU oracle of the reference algorithm -- test infrastructure only (see bagpipe_oracle.py)."""
