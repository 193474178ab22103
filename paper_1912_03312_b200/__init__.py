"""B200-native REXI time step (arXiv 1912.03312) -- placeholder, filled in below."""
