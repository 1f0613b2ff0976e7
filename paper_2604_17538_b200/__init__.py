"""B200-native XPSQ SDF + smooth contact manifolds (arXiv 2604.17538)."""
