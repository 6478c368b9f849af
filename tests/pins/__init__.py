"""Independent pins for the oracle (test code; never imported by the product path)."""
