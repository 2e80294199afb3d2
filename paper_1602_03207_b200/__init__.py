"""B200-native A-V eddy-current assembly + Krylov hot path (arXiv 1602.03207 / ectsim)."""
