"""B200-native GFlowNet training engine (gfnx hot path, arXiv 2511.16592)."""
from . import abi  # noqa: F401
