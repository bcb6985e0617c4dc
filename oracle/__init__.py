"""CPU oracle for the FHV hot path -- test infrastructure only (see fhv_oracle.c)."""
