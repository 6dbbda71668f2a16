"""B200-native D-NGD step (arXiv 2505.21404) behind the reference `dngd` API."""
