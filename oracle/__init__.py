"""CPU oracle for the CULSH-MF hot path -- test infrastructure only (see oracle.py)."""
