"""B200-native dock-and-score hot path of EXSCALATE (arXiv 2110.11644)."""
