"""TEST INFRASTRUCTURE ONLY: parity oracle (reference build + C restatement)."""
