"""CPU oracle (test infrastructure only — see covoracle.py's header)."""
