"""CPU checkers for the decode-attention path (test infrastructure only)."""
