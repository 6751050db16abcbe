"""B200-native (sm_100a) Gaussian map-optimisation hot path of Gaussian-LIC2 (arXiv 2507.04004).

Drop-in for the reference's `splatslam.rasterizer`, `splatslam.losses` and `splatslam.gaussians`
entry points (forward / backward / sparse_adam_step / mapping_loss / project / eval_sh) and
the `optimize_map` loop of `splatslam.mapper`; all compute runs in hand-written CUDA kernels
behind the C ABI of include/gslic.h.
"""

from . import errors  # noqa: F401

__all__ = ["errors", "gaussians", "rasterizer", "losses", "mapper", "scenes", "build"]
__version__ = "0.1.0"
