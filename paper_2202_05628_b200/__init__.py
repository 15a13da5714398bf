"""B200-native warp -> octree rebuild -> render hot path of the ARTEMIS
NGI-animal renderer (arXiv 2202.05628), behind the reference's `animvox`
kernel contract. See DESIGN.md."""

__version__ = "0.1.0"
