"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY (see oracle/sto_oracle.c)."""
