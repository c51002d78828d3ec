"""B200-native FCA / FastFCA EM (package init placeholder)."""
