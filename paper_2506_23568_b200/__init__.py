"""B200-native HHFFBPA / BPA hot path (placeholder; filled in below)."""
