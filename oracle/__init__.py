"""CPU oracle (test infrastructure only; see oracle/emc_oracle.c)."""
