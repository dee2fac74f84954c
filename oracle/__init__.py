"""TEST INFRASTRUCTURE ONLY: CPU oracles (compiled reference + C restatement)."""
