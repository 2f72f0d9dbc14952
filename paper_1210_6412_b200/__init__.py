"""B200-native Jacobi / BiCGStab reachability solver (arXiv 1210.6412)."""
