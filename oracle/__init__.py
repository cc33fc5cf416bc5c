"""TEST INFRASTRUCTURE ONLY: CPU checkers for the CUDA product path (see pdlp_oracle.h)."""
