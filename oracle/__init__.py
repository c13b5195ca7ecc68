"""CPU oracle (test infrastructure only; see tc_oracle.h)."""
