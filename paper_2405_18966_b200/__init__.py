"""B200-native hot path of svds-C (arXiv 2405.18966); see DESIGN.md."""
