"""B200-native decode attention for MLRA-4 / MLA / GQA (drop-in for attnkit's decode API)."""
