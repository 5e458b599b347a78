"""B200-native Stein-particle-filter step (MegaParticles, arXiv 2404.16370).

Drop-in for the reference ``steinmcl`` filter hot path: hand-written sm_100a
kernels behind the C ABI of include/smcl_gpu.h (libsmcl_gpu.so, built in-tree),
with a Python mirror of the reference API in ``api`` and the synthetic
workload generator in ``sim``.
"""
from .abi import CORRIDOR_CFG, DEFAULT_CONFIG, Particles, make_config  # noqa: F401
from .api import (FilterConfig, FilterEngine, GaussianCloud, build_nnf, downsample_to,  # noqa: F401
                  estimate_covariances, make_scan_cloud)

__all__ = ["FilterEngine", "FilterConfig", "GaussianCloud", "Particles", "make_config", "make_scan_cloud",
           "estimate_covariances", "downsample_to", "build_nnf", "DEFAULT_CONFIG", "CORRIDOR_CFG"]
