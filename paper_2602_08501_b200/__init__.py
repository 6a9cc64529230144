"""B200-native accelerator for the MP-WSD two-stage decoding hot path."""
