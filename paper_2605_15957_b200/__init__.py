"""B200-native filtered vector-search operator (arXiv 2605.15957 Vec-H)."""
