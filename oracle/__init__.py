"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference (the parity checker)."""
