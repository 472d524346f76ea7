"""B200-native multi-signal growing self-organizing network (arXiv:1503.08294)."""
