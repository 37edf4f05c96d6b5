"""CPU checkers for the MSBFM hot path -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.c)."""
