"""B200-native DeDLOC averaging round (arXiv 2106.10207), drop-in for the
swarmplan reference's strategy -> averaging path. See DESIGN.md."""
from .round import AveragingRound, fill_synthetic, part_offsets  # noqa: F401

__version__ = "0.1.0"
