"""CPU checkers for the TBIK hot path (test infrastructure only; see oracle/oracle.py)."""
