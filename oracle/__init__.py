"""CPU oracle (test infrastructure only; see oracle/port.py)."""
