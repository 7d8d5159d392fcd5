"""B200-native batched JaxLrauv environment step (arXiv 2505.08222)."""
