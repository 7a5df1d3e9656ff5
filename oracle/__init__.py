"""CPU oracle for the TAP search hot path -- test infrastructure only (see oracle.c)."""
