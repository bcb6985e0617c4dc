"""B200-native fragment-history volumes (placeholder, filled below)."""
